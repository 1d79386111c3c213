"""CPU oracle for the derived two-pass PQ search — TEST INFRASTRUCTURE ONLY.

This module restates, in numpy, the reference `derivedpq` query path
(/root/reference/pkg/src/derivedpq, v0.1.0) so that the B200 implementation
can be checked against it where /root/reference does not exist (the GPU box).
It is imported only by tests/, by __graft_entry__.smoke() as the checker,
and by bench.py's cpu_baseline / --impl reference legs.  The product path
(paper_1905_06900_b200) never imports it and fails loudly without its CUDA
library.

Parity pinning: tests/golden/*.npz hold outputs of the reference itself,
generated in the build container by tests/golden/make_golden.py (which
imports /root/reference); tests/test_oracle_golden.py checks this restatement
against them bit-for-bit, so the oracle is pinned, not merely plausible.

Each function names the reference lines it follows.  The arithmetic (dtype
of every intermediate, summation order) is kept identical on purpose: the
B200 kernels must reproduce these bits.
"""

from __future__ import annotations

import time

import numpy as np

SATURATED = 255  # twopass.py:184


# ---------------------------------------------------------------- tables --

def sq_dist_rows(rows: np.ndarray, v: np.ndarray) -> np.ndarray:
    """search.py:16-25 row_sq_dists: f32 diff, f32 square, numpy row sum."""
    diff = rows - v
    return (diff * diff).sum(axis=1)


def lookup_tables(y: np.ndarray, codebooks: np.ndarray) -> np.ndarray:
    """search.py:28-48 compute_tables: (m, k) f32 distances of y's sub-vectors."""
    m, k, dsub = codebooks.shape
    y = np.asarray(y, dtype=np.float32).reshape(-1)
    if y.size != m * dsub:
        raise ValueError(f"query dimension {y.size} != {m}*{dsub}")
    parts = y.reshape(m, dsub)
    out = np.empty((m, k), dtype=np.float32)
    for j in range(m):
        out[j] = sq_dist_rows(codebooks[j], parts[j])
    return out


def table_sums(codes: np.ndarray, tables: np.ndarray) -> np.ndarray:
    """search.py:64-70 adc_batch: f64 accumulation in subspace order."""
    total = np.zeros(codes.shape[0], dtype=np.float64)
    for j in range(tables.shape[0]):
        total += tables[j, codes[:, j]]
    return total


def best_r(dists: np.ndarray, ids: np.ndarray, r: int):
    """search.py:73-88 top_r_by_distance: ascending (dist, id), exact ties."""
    n = dists.shape[0]
    if r >= n:
        order = np.lexsort((ids, dists))
        return ids[order], dists[order]
    part = np.argpartition(dists, r - 1)[:r]
    cut = dists[part].max()
    keep = np.flatnonzero(dists <= cut)
    order = keep[np.lexsort((ids[keep], dists[keep]))][:r]
    return ids[order], dists[order]


# ----------------------------------------------------- 8-bit quantization --

class Quantized:
    """twopass.py:26-38 QuantizedTables (q u8 (m,kbar), qmin, qmax, bbar)."""

    __slots__ = ("q", "qmin", "qmax", "bbar")

    def __init__(self, q, qmin, qmax, bbar):
        self.q, self.qmin, self.qmax, self.bbar = q, qmin, qmax, bbar


def low_float_scores(codes: np.ndarray, small: np.ndarray, bbar: int) -> np.ndarray:
    """twopass.py:41-47 _adc_low_float: masked gather, f64 sum, j ascending."""
    mask = (1 << bbar) - 1
    total = np.zeros(codes.shape[0], dtype=np.float64)
    for j in range(small.shape[0]):
        total += small[j, codes[:, j] & mask]
    return total


def quantize_bounded(small: np.ndarray, qmin: float, qmax: float, bbar: int) -> Quantized:
    """twopass.py:50-60 quantize_with_bounds.

    f64 formula, clip to [0, 254], then 255 where small > qmax — the
    comparison of an f32 array with a Python float runs in f32 (NEP 50).
    """
    if qmax <= qmin:
        return Quantized(np.zeros(small.shape, dtype=np.uint8), qmin, qmin, bbar)
    scale = 255.0 / (qmax - qmin)
    q = np.clip(np.floor((small.astype(np.float64) - qmin) * scale), 0, 254).astype(np.uint8)
    q[small > qmax] = SATURATED
    return Quantized(q, qmin, qmax, bbar)


def quantize_small(small: np.ndarray, prefix_codes: np.ndarray, r2: int) -> Quantized:
    """twopass.py:63-85 quantize_tables: qmin over all entries, qmax = max
    float score of the first min(r2, len) prefix codes."""
    prefix_codes = np.asarray(prefix_codes)
    if prefix_codes.shape[0] == 0:
        raise ValueError("need at least one code to estimate qmax")
    kbar = small.shape[1]
    bbar = int(kbar).bit_length() - 1
    if kbar != (1 << bbar):
        raise ValueError(f"small table size {kbar} is not a power of two")
    qmin = float(small.min())
    lead = prefix_codes[: min(r2, len(prefix_codes))]
    qmax = float(low_float_scores(lead, small, bbar).max())
    return quantize_bounded(small, qmin, qmax, bbar)


def low_scores(codes: np.ndarray, qt: Quantized) -> np.ndarray:
    """twopass.py:99-106 adc_low_batch: int32 masked sum, saturate at 255."""
    mask = (1 << qt.bbar) - 1
    acc = qt.q[0, codes[:, 0] & mask].astype(np.int32)
    for j in range(1, qt.q.shape[0]):
        acc += qt.q[j, codes[:, j] & mask]
    return np.minimum(acc, SATURATED).astype(np.uint8)


# ------------------------------------------------------ bucketed selection --

def bucket_bound(scores: np.ndarray, r2: int, capped: bool = True) -> int:
    """twopass.py:171-186 CappedBuckets.from_arrays bound: 255 (keep all
    live) unless the live count reaches r2, then searchsorted(cum, r2)+1."""
    if r2 < 1:
        raise ValueError(f"r2 must be >= 1, got {r2}")
    counts = np.bincount(scores, minlength=256)[:SATURATED].astype(np.int64)
    bound = SATURATED
    if capped:
        cum = np.cumsum(counts)
        if cum[-1] >= r2:
            bound = int(np.searchsorted(cum, r2)) + 1
    return bound


def bucket_walk(scores: np.ndarray, ids: np.ndarray, r2: int, capped: bool = True) -> np.ndarray:
    """Candidate ids the refine pass scores.

    twopass.py:187-200 keeps scores < bound, stable-sorted into buckets;
    twopass.py:295-302 walks buckets in ascending order taking whole
    buckets until at least r2 ids are taken.  Returned in walk order."""
    scores = np.asarray(scores)
    ids = np.asarray(ids)
    if scores.shape[0] == 0:
        return np.empty(0, dtype=np.int64)
    bound = bucket_bound(scores, r2, capped)
    live = scores < bound
    s_live = scores[live]
    i_live = ids[live]
    order = np.argsort(s_live, kind="stable")
    s_sorted = s_live[order]
    i_sorted = i_live[order]
    taken = 0
    end = 0
    for b in range(bound):
        hi = int(np.searchsorted(s_sorted, b, side="right"))
        if hi > end:
            taken += hi - end
            end = hi
            if taken >= r2:
                break
    return np.asarray(i_sorted[:end], dtype=np.int64)


def closed_form_bstar(scores: np.ndarray, r2: int) -> int:
    """SURVEY Appendix A rule 8: b* = min{b : #(s <= b, s < 255) >= r2},
    else 254.  Equal to the walk above (checked by tests)."""
    counts = np.bincount(scores, minlength=256)[:SATURATED]
    cum = np.cumsum(counts)
    hit = np.flatnonzero(cum >= r2)
    return int(hit[0]) if hit.size else 254


# ----------------------------------------------------------- lazy refine --

class LazyFull:
    """twopass.py:220-251 LazyTables: sentinel -1, fill on demand with the
    same row kernel as eager tables (bit-identical entries)."""

    def __init__(self, codebooks: np.ndarray, y: np.ndarray):
        m, k, dsub = codebooks.shape
        y = np.asarray(y, dtype=np.float32).reshape(-1)
        if y.size != m * dsub:
            raise ValueError(f"query dimension {y.size} != {m}*{dsub}")
        self.codebooks = codebooks
        self.parts = y.reshape(m, dsub)
        self.tables = np.full((m, k), -1.0, dtype=np.float32)
        self.n_computed = 0

    def fill(self, j: int, idx: np.ndarray) -> None:
        idx = np.unique(idx)
        todo = idx[self.tables[j, idx] == -1.0]
        if todo.size:
            self.tables[j, todo] = sq_dist_rows(self.codebooks[j][todo], self.parts[j])
            self.n_computed += int(todo.size)

    def score(self, codes: np.ndarray) -> np.ndarray:
        """twopass.py:269-273 _refine_batch."""
        for j in range(codes.shape[1]):
            self.fill(j, codes[:, j])
        return table_sums(codes, self.tables)


# ---------------------------------------------------------- one query --

def derived_one(codebooks, derived, rotate, codes, y, r, r2, capped=True):
    """twopass.py:311-353 nns_derived for one query.

    Returns (ids, dists, info) with ids/dists sorted by (dist, id) and info
    holding the intermediates the GPU debug seams expose."""
    if r > r2:
        raise ValueError(f"r={r} must not exceed r2={r2}")
    codes = np.asarray(codes)
    y = np.asarray(y, dtype=np.float32).reshape(-1)
    yr = rotate(y.reshape(1, -1)).reshape(-1)
    t0 = time.perf_counter_ns()
    small = lookup_tables(yr, derived)
    qt = quantize_small(small, codes[: min(r2, codes.shape[0])], r2)
    t1 = time.perf_counter_ns()
    rows = np.arange(codes.shape[0], dtype=np.int64)
    scores = low_scores(codes, qt) if codes.shape[0] else np.empty(0, np.uint8)
    cand = bucket_walk(scores, rows, r2, capped)
    t2 = time.perf_counter_ns()
    if cand.size:
        lazy = LazyFull(codebooks, yr)
        dists = lazy.score(codes[cand])
        ids, ds = best_r(dists, cand, r)
    else:
        ids, ds = np.empty(0, np.int64), np.empty(0, np.float64)
    t3 = time.perf_counter_ns()
    info = {"small": small, "q": qt.q, "qmin": qt.qmin, "qmax": qt.qmax,
            "scores": scores, "ncand": int(cand.size),
            "tables_us": (t1 - t0) / 1e3, "scan_us": (t2 - t1) / 1e3, "refine_us": (t3 - t2) / 1e3}
    return ids, ds, info


def conventional_one(codebooks, rotate, codes, y, r):
    """flat.py:82-93: full tables, table sums over every code, top-r."""
    yr = rotate(np.asarray(y, dtype=np.float32).reshape(1, -1)).reshape(-1)
    tables = lookup_tables(yr, codebooks)
    dists = table_sums(codes, tables)
    return best_r(dists, np.arange(codes.shape[0], dtype=np.int64), r)


def pack(rows, r: int):
    """flat.py:16-29 pack_results: (nq, r) f64 +inf-padded, i64 -1-padded."""
    nq = len(rows)
    dists = np.full((nq, r), np.inf, dtype=np.float64)
    ids = np.full((nq, r), -1, dtype=np.int64)
    for qi, (i, d) in enumerate(rows):
        got = len(i)
        if got:
            dists[qi, :got] = d
            ids[qi, :got] = i
    return dists, ids


def identity_rotate(x):
    return x


def make_rotate(rotation):
    """quantizer.py:235-239 rotate: (X @ R) in f32, identity when None."""
    if rotation is None:
        return identity_rotate
    return lambda x: (x @ rotation).astype(np.float32, copy=False)


def flat_search(codebooks, derived, codes, Y, r, mode="conventional", r2=None,
                capped=True, rotation=None):
    """flat.py:54-108 FlatIndex.search (results only)."""
    Y = np.ascontiguousarray(Y, dtype=np.float32)
    rot = make_rotate(rotation)
    rows = []
    if mode == "conventional":
        for qi in range(Y.shape[0]):
            rows.append(conventional_one(codebooks, rot, codes, Y[qi], r))
    elif mode == "derived":
        if r2 is None:
            raise ValueError("derived mode requires r2")
        for qi in range(Y.shape[0]):
            ids, ds, _ = derived_one(codebooks, derived, rot, codes, Y[qi], r, r2, capped)
            rows.append((ids, ds))
    else:
        raise ValueError(f"unknown mode {mode!r}")
    return pack(rows, r)


# ----------------------------------------------------------------- IVF --

def ivf_probe(centers: np.ndarray, y: np.ndarray, ma: int):
    """ivf.py:107-120 probe: f64 einsum distances, top-ma, lower id on ties;
    residuals y - center in f32."""
    n_cells = centers.shape[0]
    y = np.asarray(y, dtype=np.float32).reshape(-1)
    if not (1 <= ma <= n_cells):
        raise ValueError(f"ma must be in [1, {n_cells}], got {ma}")
    diff = centers.astype(np.float64) - y.astype(np.float64)
    d2 = np.einsum("kd,kd->k", diff, diff)
    cells, _ = best_r(d2, np.arange(n_cells, dtype=np.int64), ma)
    return cells, y[None, :] - centers[cells]


def ivf_derived_one(ivf, y, r, r2, ma, capped=True):
    """ivf.py:195-277 _search_derived for one query.

    `ivf` is a mapping/object with centers, offsets, sorted_codes,
    sorted_ids, cell_of, row_of, codebooks, derived, bbar, rotate."""
    cells, res = ivf_probe(ivf["centers"], y, ma)
    rotated = ivf["rotate"](res)
    off = ivf["offsets"]
    qts = {}
    bounds = None
    for ci, cell in enumerate(cells):
        lo, hi = int(off[cell]), int(off[cell + 1])
        if lo == hi:
            continue
        small = lookup_tables(rotated[ci], ivf["derived"])
        if bounds is None:
            qt = quantize_small(small, ivf["sorted_codes"][lo: lo + min(r2, hi - lo)], r2)
            bounds = (qt.qmin, qt.qmax)
        else:
            qt = quantize_bounded(small, bounds[0], bounds[1], ivf["bbar"])
        qts[int(cell)] = qt
    score_parts, id_parts = [], []
    for cell in cells:
        lo, hi = int(off[cell]), int(off[cell + 1])
        if lo == hi:
            continue
        score_parts.append(low_scores(ivf["sorted_codes"][lo:hi], qts[int(cell)]))
        id_parts.append(ivf["sorted_ids"][lo:hi])
    if not score_parts:
        return np.empty(0, np.int64), np.empty(0, np.float64), {"ncand": 0, "bounds": None}
    cand = bucket_walk(np.concatenate(score_parts), np.concatenate(id_parts), r2, capped)
    if cand.size == 0:
        return np.empty(0, np.int64), np.empty(0, np.float64), {"ncand": 0, "bounds": bounds}
    frame = {int(c): rotated[ci] for ci, c in enumerate(cells)}
    cand_cells = ivf["cell_of"][cand]
    d_parts, i_parts = [], []
    for cell in np.unique(cand_cells):
        members = cand[cand_cells == cell]
        lazy = LazyFull(ivf["codebooks"], frame[int(cell)])
        d_parts.append(lazy.score(ivf["sorted_codes"][ivf["row_of"][members]]))
        i_parts.append(members)
    ids, ds = best_r(np.concatenate(d_parts), np.concatenate(i_parts), r)
    return ids, ds, {"ncand": int(cand.size), "bounds": bounds}


def ivf_conventional_one(ivf, y, r, ma):
    """ivf.py:162-193 _search_conventional for one query."""
    cells, res = ivf_probe(ivf["centers"], y, ma)
    rotated = ivf["rotate"](res)
    off = ivf["offsets"]
    d_parts, i_parts = [], []
    for ci, cell in enumerate(cells):
        lo, hi = int(off[cell]), int(off[cell + 1])
        if lo == hi:
            continue
        tables = lookup_tables(rotated[ci], ivf["codebooks"])
        d_parts.append(table_sums(ivf["sorted_codes"][lo:hi], tables))
        i_parts.append(ivf["sorted_ids"][lo:hi])
    if not d_parts:
        return np.empty(0, np.int64), np.empty(0, np.float64)
    return best_r(np.concatenate(d_parts), np.concatenate(i_parts), r)


def ivf_search(ivf, Y, r, ma=8, mode="conventional", r2=None, capped=True):
    """ivf.py:125-160 IVFIndex.search (results only)."""
    Y = np.ascontiguousarray(Y, dtype=np.float32)
    if mode not in ("conventional", "derived"):
        raise ValueError(f"unknown mode {mode!r}")
    if mode == "derived":
        if r2 is None:
            raise ValueError("derived mode requires r2")
        if r > r2:
            raise ValueError(f"r={r} must not exceed r2={r2}")
    rows = []
    for qi in range(Y.shape[0]):
        if mode == "conventional":
            rows.append(ivf_conventional_one(ivf, Y[qi], r, ma))
        else:
            ids, ds, _ = ivf_derived_one(ivf, Y[qi], r, r2, ma, capped)
            rows.append((ids, ds))
    return pack(rows, r)


# ----------------------------------------------------------- evaluation --

def exact_nn(database, queries, depth: int) -> np.ndarray:
    """evaluation.py:28-62: brute force in f64, ties to the lower id."""
    db = np.ascontiguousarray(database, dtype=np.float32).astype(np.float64)
    qs = np.ascontiguousarray(queries, dtype=np.float32)
    n = db.shape[0]
    depth = min(depth, n)
    norms = np.einsum("nd,nd->n", db, db)
    ids = np.arange(n, dtype=np.int64)
    out = np.empty((qs.shape[0], depth), dtype=np.int32)
    step = max(1, (2 ** 25) // max(n, 1))
    for s in range(0, qs.shape[0], step):
        blk = qs[s: s + step].astype(np.float64)
        d2 = norms[None, :] - 2.0 * (blk @ db.T)
        d2 += np.einsum("qd,qd->q", blk, blk)[:, None]
        for i in range(d2.shape[0]):
            out[s + i] = best_r(d2[i], ids, depth)[0]
    return out


def recall_at_r(ids: np.ndarray, truth: np.ndarray, r: int) -> float:
    """evaluation.py:76-92: fraction of queries whose rank-0 true neighbour
    is among the first r results."""
    ids = np.asarray(ids)
    truth = np.asarray(truth)
    return float((ids[:, :r] == truth[:, :1]).any(axis=1).mean())
