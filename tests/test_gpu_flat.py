"""Parity of the CUDA flat path (libdpq.so through the C ABI) with the
reference (golden fixtures) and with the CPU oracle on seeded inputs.

Bar: bit-exact.  Small tables, 8-bit tables, qmin/qmax, candidate counts,
result ids and f64 distances must equal the reference's bits; the
north_star tolerance (1e-4 relative) is therefore met with margin 0.
"""

import os

import numpy as np
import pytest

from conftest import FLAT_CASES, load_golden
from oracle import derived_search as O
from paper_1905_06900_b200 import datagen
from paper_1905_06900_b200.flat import FlatIndex

pytestmark = pytest.mark.gpu


def _index(g):
    return FlatIndex.from_arrays(g["codebooks"], g["derived"], g["codes"], rotation=g.get("rotation"))


def _same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))


@pytest.mark.parametrize("name", FLAT_CASES)
def test_quantized_tables_bitwise_vs_reference(name):
    g = load_golden(name)
    idx = _index(g)
    small, q, qmin, qmax = idx.quantized_tables(g["queries"], g["meta"]["r2"])
    assert np.array_equal(small.view(np.uint32), g["exp_small"].view(np.uint32))
    assert np.array_equal(q, g["exp_q"])
    assert np.array_equal(qmin, g["exp_qmin"]) and np.array_equal(qmax, g["exp_qmax"])


@pytest.mark.parametrize("name", FLAT_CASES)
def test_candidate_counts_vs_reference(name):
    g = load_golden(name)
    _, ncand = _index(g).candidate_counts(g["queries"], g["meta"]["r2"])
    assert np.array_equal(ncand, g["exp_ncand"])


@pytest.mark.parametrize("name", FLAT_CASES)
def test_derived_search_bitwise_vs_reference(name):
    g = load_golden(name)
    m = g["meta"]
    d, i = _index(g).search(g["queries"], m["r"], mode="derived", r2=m["r2"])
    assert np.array_equal(i, g["exp_derived_i"])
    assert _same(d, g["exp_derived_d"])
    d2, i2 = _index(g).search(g["queries"], m["r"], mode="derived", r2=m["r2"], capped=False)
    assert np.array_equal(i2, i) and _same(d2, d)


@pytest.mark.parametrize("name", FLAT_CASES)
def test_conventional_and_full_budget_vs_reference(name):
    g = load_golden(name)
    idx = _index(g)
    if "exp_conv_i" in g:
        d, i = idx.search(g["queries"], g["meta"]["r"])
        assert np.array_equal(i, g["exp_conv_i"]) and _same(d, g["exp_conv_d"])
    if "exp_full_i" in g:
        r = g["exp_full_i"].shape[1]
        d, i = idx.search(g["queries"][:4], r, mode="derived", r2=len(g["codes"]), capped=False)
        assert np.array_equal(i, g["exp_full_i"]) and _same(d, g["exp_full_d"])


def test_config1_shape_bitwise_vs_reference(c1_golden):
    """PQ 4x16 / derived 4x8, N=100k, Q=100, r2=1000, k=100 (config 1)."""
    g = c1_golden
    idx = FlatIndex.from_arrays(g["codebooks"], g["derived"], g["codes"])
    small, q, qmin, qmax = idx.quantized_tables(g["queries"], 1000)
    assert np.array_equal(q, g["exp_q"]) and np.array_equal(qmax, g["exp_qmax"])
    _, ncand = idx.candidate_counts(g["queries"], 1000)
    assert np.array_equal(ncand, g["exp_ncand"])
    d, i = idx.search(g["queries"], 100, mode="derived", r2=1000)
    assert np.array_equal(i, g["exp_derived_i"])
    assert _same(d, g["exp_derived_d"])


# ------------------------------------------------------ seeded vs oracle --

def _model(rng, m, k, kbar, dsub):
    """Random valid model: full codebook rows, derived = group means over
    the low-bit groups (so low bits index the derived codebook)."""
    cb = rng.normal(size=(m, k, dsub)).astype(np.float32) * 3
    der = np.stack([np.stack([cb[j][np.arange(k) % kbar == g].mean(axis=0) for g in range(kbar)])
                    for j in range(m)]).astype(np.float32)
    return cb, der


def _encode(cb, X):
    m, k, dsub = cb.shape
    out = np.empty((X.shape[0], m), np.uint16 if k > 256 else np.uint8)
    for j in range(m):
        sub = X[:, j * dsub:(j + 1) * dsub].astype(np.float64)
        c = cb[j].astype(np.float64)
        d2 = (sub * sub).sum(1)[:, None] - 2 * sub @ c.T + (c * c).sum(1)[None, :]
        out[:, j] = d2.argmin(1)
    return out


def _oracle(cb, der, codes, Y, r, r2):
    return O.flat_search(cb, der, codes, Y, r, "derived", r2)


CASES = [
    # m, k, kbar, dsub, n, nq, r, r2
    (4, 256, 16, 8, 5000, 40, 10, 300),
    (1, 64, 8, 4, 3000, 9, 5, 50),
    (3, 512, 32, 6, 4000, 70, 20, 400),
    (5, 256, 64, 3, 3000, 33, 7, 100),
    (8, 256, 256, 4, 3000, 20, 10, 250),
    (2, 1024, 256, 16, 6000, 130, 100, 1000),
    (4, 4096, 256, 32, 20000, 65, 100, 1000),
    (6, 128, 8, 7, 2000, 12, 3, 3),
]


@pytest.mark.parametrize("case", CASES)
def test_seeded_random_models_vs_oracle(case):
    m, k, kbar, dsub, n, nq, r, r2 = case
    rng = np.random.default_rng(hash(case) % 2**32)
    cb, der = _model(rng, m, k, kbar, dsub)
    X = (cb[np.arange(m)[None, :], rng.integers(0, k, size=(n, m))].reshape(n, m * dsub)
         + rng.normal(scale=0.5, size=(n, m * dsub))).astype(np.float32)
    codes = _encode(cb, X)
    Y = (X[rng.integers(0, n, size=nq)] + rng.normal(scale=0.3, size=(nq, m * dsub))).astype(np.float32)
    d0, i0 = _oracle(cb, der, codes, Y, r, r2)
    d1, i1 = FlatIndex.from_arrays(cb, der, codes).search(Y, r, mode="derived", r2=r2)
    assert np.array_equal(i0, i1)
    assert _same(d0, d1)


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("case", CASES)
def test_seeded_random_models_more_seeds(case, seed):
    """More seeds of the same shapes, plus single-query searches against the
    batched ones (batch invariance at small sizes, padding-heavy tiles)."""
    m, k, kbar, dsub, n, nq, r, r2 = case
    rng = np.random.default_rng(seed * 7919 + CASES.index(case))
    cb, der = _model(rng, m, k, kbar, dsub)
    X = (cb[np.arange(m)[None, :], rng.integers(0, k, size=(n, m))].reshape(n, m * dsub)
         + rng.normal(scale=0.5, size=(n, m * dsub))).astype(np.float32)
    codes = _encode(cb, X)
    Y = (X[rng.integers(0, n, size=nq)] + rng.normal(scale=0.3, size=(nq, m * dsub))).astype(np.float32)
    d0, i0 = _oracle(cb, der, codes, Y, r, r2)
    idx = FlatIndex.from_arrays(cb, der, codes)
    d1, i1 = idx.search(Y, r, mode="derived", r2=r2)
    assert np.array_equal(i0, i1) and _same(d0, d1)
    for qi in range(min(nq, 3)):
        d2, i2 = idx.search(Y[qi:qi + 1], r, mode="derived", r2=r2)
        assert np.array_equal(i2[0], i0[qi]) and _same(d2[0], d0[qi])


def test_edge_cases_vs_oracle():
    rng = np.random.default_rng(7)
    cb, der = _model(rng, 4, 256, 16, 4)
    # N=1; r2 > N; r > N (padding)
    for n, r, r2 in [(1, 1, 1), (1, 5, 10), (7, 10, 50), (300, 300, 300), (300, 50, 5000)]:
        codes = rng.integers(0, 256, size=(n, 4)).astype(np.uint8)
        Y = rng.normal(size=(5, 16)).astype(np.float32) * 3
        d0, i0 = _oracle(cb, der, codes, Y, r, r2)
        d1, i1 = FlatIndex.from_arrays(cb, der, codes).search(Y, r, mode="derived", r2=r2)
        assert np.array_equal(i0, i1) and _same(d0, d1), (n, r, r2)
    # all codes identical: qmax == qmin (degenerate zeros), every row refined,
    # all distances tie -> ids ascending
    codes = np.tile(rng.integers(0, 256, size=(1, 4)), (500, 1)).astype(np.uint8)
    Y = rng.normal(size=(4, 16)).astype(np.float32)
    d0, i0 = _oracle(cb, der, codes, Y, 20, 10 + 20)
    d1, i1 = FlatIndex.from_arrays(cb, der, codes).search(Y, 20, mode="derived", r2=30)
    assert np.array_equal(i0, i1) and _same(d0, d1)
    assert np.array_equal(i1[0], np.arange(20))
    # many duplicate codes: (dist, id) tie-breaking inside the top-r
    codes = rng.integers(0, 4, size=(2000, 4)).astype(np.uint8)
    d0, i0 = _oracle(cb, der, codes, Y, 50, 200)
    d1, i1 = FlatIndex.from_arrays(cb, der, codes).search(Y, 50, mode="derived", r2=200)
    assert np.array_equal(i0, i1) and _same(d0, d1)


def _sift_setup(n, nq, seed=3, k=4096):
    st = datagen.seed_streams(seed)
    centres = datagen.sift_centres(st["centres"])
    X = datagen.sift_like(st["database"], centres, n)
    Y = datagen.sift_like(st["queries"], centres, nq)
    rng = np.random.default_rng(seed)
    cb = np.stack([X[rng.choice(n, size=k, replace=False), j * 32:(j + 1) * 32] for j in range(4)])
    der = np.stack([np.stack([cb[j][np.arange(k) % 256 == g].mean(axis=0) for g in range(256)])
                    for j in range(4)]).astype(np.float32)
    codes = rng.integers(0, k, size=(n, 4)).astype(np.uint16)
    return cb.astype(np.float32), der, codes, Y


def test_sampled_guard_path_vs_oracle():
    """N above the exact-histogram limit: the guard comes from a row sample."""
    cb, der, codes, Y = _sift_setup(200_000, 6)
    d0, i0 = _oracle(cb, der, codes, Y, 100, 1000)
    idx = FlatIndex.from_arrays(cb, der, codes)
    d1, i1 = idx.search(Y, 100, mode="derived", r2=1000)
    assert np.array_equal(i0, i1) and _same(d0, d1)


def test_forced_exact_redo_and_overflow(monkeypatch):
    """Tiny guard sample (guards too tight -> exact redo) and a tiny emit
    capacity (overflow -> grow and rerun) still give the exact answer."""
    cb, der, codes, Y = _sift_setup(120_000, 5, seed=4)
    d0, i0 = _oracle(cb, der, codes, Y, 50, 800)
    monkeypatch.setenv("DPQ_GUARD_SAMPLE", "16")
    monkeypatch.setenv("DPQ_EXACT_LIMIT", "0")
    monkeypatch.setenv("DPQ_EMIT_CAP", "32")
    idx = FlatIndex.from_arrays(cb, der, codes)
    d1, i1 = idx.search(Y, 50, mode="derived", r2=800)
    assert np.array_equal(i0, i1) and _same(d0, d1)
    assert idx._handle().counters()["fallbacks"] > 0


def test_batch_invariance():
    g = load_golden("pq_blobs")
    idx = _index(g)
    ref = idx.search(g["queries"], 10, mode="derived", r2=300)
    for b in (1, 5, 64, 1024):
        idx._handle().set_batch(b)
        d, i = idx.search(g["queries"], 10, mode="derived", r2=300)
        assert np.array_equal(i, ref[1]) and _same(d, ref[0])


def test_timings_and_errors():
    g = load_golden("pq_blobs")
    idx = _index(g)
    _, _, t = idx.search(g["queries"][:3], 5, mode="derived", r2=100, return_timings=True)
    assert set(t) == {"index_us", "tables_us", "scan_us", "refine_us"}
    assert np.all(t["index_us"] == 0.0) and np.all(t["refine_us"] > 0.0)
    _, _, t = idx.search(g["queries"][:3], 5, return_timings=True)
    assert np.all(t["refine_us"] == 0.0)
    with pytest.raises(ValueError, match="must not exceed"):
        idx.search(g["queries"], 11, mode="derived", r2=10)
    with pytest.raises(ValueError, match="r2"):
        idx.search(g["queries"], 5, mode="derived")
    with pytest.raises(ValueError, match="mode"):
        idx.search(g["queries"], 5, mode="hybrid")
    dists, ids = idx.search(g["queries"][:1], len(g["codes"]) + 10)
    assert (ids[0] >= 0).sum() == len(g["codes"]) and np.isinf(dists[0, len(g["codes"]):]).all()


def test_seven_bit_fast_tiles_vs_oracle():
    """Small r2 over a larger database puts every guard <= 126, so every tile
    takes the clamped 7-bit scan path; results must stay bit-exact."""
    cb, der, codes, Y = _sift_setup(150_000, 40, seed=8)
    idx = FlatIndex.from_arrays(cb, der, codes)
    bstar, _ = idx.candidate_counts(Y, 60)
    assert bstar.max() <= 120, bstar.max()
    d0, i0 = _oracle(cb, der, codes, Y, 20, 60)
    d1, i1 = idx.search(Y, 20, mode="derived", r2=60)
    assert np.array_equal(i0, i1) and _same(d0, d1)
    # and a mixed batch: half the tile with large r2 guards (not clamped)
    d0, i0 = _oracle(cb, der, codes, Y[:8], 20, 3000)
    d1, i1 = idx.search(Y[:8], 20, mode="derived", r2=3000)
    assert np.array_equal(i0, i1) and _same(d0, d1)


@pytest.mark.parametrize("r2", [20, 150, 1200])
def test_wide_tiles_vs_oracle(r2, monkeypatch):
    """Guards <= 62 put tiles in the wide 5/6-bit scan loop (16 queries per
    lane, bias folded into subspace 0 for 5-bit tiles).  Bit-exact against
    the oracle, and identical to the scan with the wide loop disabled."""
    cb, der, codes, Y = _sift_setup(150_000, 40, seed=11)
    idx = FlatIndex.from_arrays(cb, der, codes)
    bstar, _ = idx.candidate_counts(Y, r2)
    d0, i0 = _oracle(cb, der, codes, Y, 20, r2)
    d1, i1 = idx.search(Y, 20, mode="derived", r2=r2)
    assert np.array_equal(i0, i1) and _same(d0, d1)
    wide = idx._handle().counters()["wide_units"]
    if bstar.max() <= 50:  # guards near b*: every tile fits 6 bits
        assert wide > 0, (bstar.max(), wide)
    monkeypatch.setenv("DPQ_SCAN_WIDE", "0")
    idx2 = FlatIndex.from_arrays(cb, der, codes)
    d2, i2 = idx2.search(Y, 20, mode="derived", r2=r2)
    assert np.array_equal(i2, i1) and _same(d2, d1)
    assert idx2._handle().counters()["wide_units"] == 0


def test_wide_tiles_mixed_guards_and_padding():
    """Batch sizes that leave padded slots in the last tile, and queries whose
    guards differ by tile mode (5-bit, 6-bit, 7-bit, generic) in one batch."""
    cb, der, codes, Y = _sift_setup(100_000, 130, seed=12)
    idx = FlatIndex.from_arrays(cb, der, codes)
    for nq, r2 in ((1, 30), (33, 100), (130, 400), (130, 5000)):
        d0, i0 = _oracle(cb, der, codes, Y[:nq], 10, r2)
        d1, i1 = idx.search(Y[:nq], 10, mode="derived", r2=r2)
        assert np.array_equal(i0, i1) and _same(d0, d1), (nq, r2)


def test_guard_sorted_slots_match_unsorted(monkeypatch):
    """Query tiles ordered by guard (flat batches) give the same results as
    the identity slot order, including a partial last tile."""
    cb, der, codes, Y = _sift_setup(120_000, 200, seed=13)
    idx = FlatIndex.from_arrays(cb, der, codes)
    d1, i1 = idx.search(Y, 15, mode="derived", r2=300)
    monkeypatch.setenv("DPQ_SORT_SLOTS", "0")
    idx2 = FlatIndex.from_arrays(cb, der, codes)
    d2, i2 = idx2.search(Y, 15, mode="derived", r2=300)
    assert np.array_equal(i1, i2) and _same(d1, d2)
    d0, i0 = _oracle(cb, der, codes, Y[:40], 15, 300)
    assert np.array_equal(i0, i1[:40]) and _same(d0, d1[:40])


def test_sorted_rows_ties_and_ids(monkeypatch):
    """The flat index stores rows sorted by (g0, g1); ids, (dist, id) tie
    order, the qmax prefix (first r2 rows in insertion order) and the
    conventional path are unchanged.  Duplicated rows force exact ties."""
    cb, der, codes, Y = _sift_setup(60_000, 12, seed=14)
    rng = np.random.default_rng(14)
    codes[rng.choice(60_000, 20_000, replace=False)] = codes[rng.integers(0, 500, 20_000)]
    d0, i0 = _oracle(cb, der, codes, Y, 40, 500)
    idx = FlatIndex.from_arrays(cb, der, codes)
    d1, i1 = idx.search(Y, 40, mode="derived", r2=500)
    assert np.array_equal(i0, i1) and _same(d0, d1)
    dc, ic = idx.search(Y[:3], 40)
    monkeypatch.setenv("DPQ_SORT_ROWS", "0")
    idx2 = FlatIndex.from_arrays(cb, der, codes)
    d2, i2 = idx2.search(Y, 40, mode="derived", r2=500)
    assert np.array_equal(i2, i1) and _same(d2, d1)
    dc2, ic2 = idx2.search(Y[:3], 40)
    assert np.array_equal(ic, ic2) and _same(dc, dc2)
    b1, n1 = idx.candidate_counts(Y, 500)
    b2, n2 = idx2.candidate_counts(Y, 500)
    assert np.array_equal(b1, b2) and np.array_equal(n1, n2)


def test_run_filter_on_encoded_data_vs_oracle(monkeypatch):
    """Rows encoded with a trained model (so (g0, g1) runs are skewed and the
    per-tile run filter skips most chunks): identical to the unfiltered scan
    and to the oracle; rows_scanned shows the filter at work."""
    import torch
    from paper_1905_06900_b200 import train

    st = datagen.seed_streams(21)
    centres = datagen.sift_centres(st["centres"])
    X = datagen.sift_like(st["database"], centres, 120_000)
    Y = datagen.sift_like(st["queries"], centres, 150)
    xt = torch.as_tensor(X, device="cuda")
    cb, der = train.train_pq(xt, 4, 12, 4, iters=8, seed=21)  # kbar = 16: 256 keys, long runs
    codes = train.encode(xt, cb).cpu().numpy().astype(np.uint16)
    idx = FlatIndex.from_arrays(cb, der, codes)
    idx.search(Y[:6], 25, mode="derived", r2=100)  # a small tile: most runs out of reach
    scanned = idx._handle().counters()["rows_scanned"]
    d1, i1 = idx.search(Y, 25, mode="derived", r2=100)
    monkeypatch.setenv("DPQ_RUN_FILTER", "0")
    idx2 = FlatIndex.from_arrays(cb, der, codes)
    idx2.search(Y[:6], 25, mode="derived", r2=100)
    assert scanned < idx2._handle().counters()["rows_scanned"] == 6 * len(codes)
    d2, i2 = idx2.search(Y, 25, mode="derived", r2=100)
    assert np.array_equal(i1, i2) and _same(d1, d2)
    d0, i0 = _oracle(cb, der, codes, Y[:30], 25, 100)
    assert np.array_equal(i0, i1[:30]) and _same(d0, d1[:30])


def test_graph_replay_and_speculation_match_eager(monkeypatch):
    """Repeated batches replay a captured CUDA graph of the speculative first
    pass; results equal the eager, non-speculative pipeline bit for bit, and a
    batch whose speculative pass is flagged (tiny guard sample -> exact redo)
    is redone exactly."""
    cb, der, codes, Y = _sift_setup(90_000, 64, seed=15)
    idx = FlatIndex.from_arrays(cb, der, codes)
    outs = [idx.search(Y, 12, mode="derived", r2=200) for _ in range(4)]  # eager, capture, replay, replay
    for d, i in outs[1:]:
        assert np.array_equal(i, outs[0][1]) and _same(d, outs[0][0])
    monkeypatch.setenv("DPQ_GRAPH", "0")
    monkeypatch.setenv("DPQ_SPECULATE", "0")
    idx2 = FlatIndex.from_arrays(cb, der, codes)
    d2, i2 = idx2.search(Y, 12, mode="derived", r2=200)
    assert np.array_equal(i2, outs[0][1]) and _same(d2, outs[0][0])
    monkeypatch.delenv("DPQ_GRAPH")
    monkeypatch.delenv("DPQ_SPECULATE")
    monkeypatch.setenv("DPQ_GUARD_SAMPLE", "8")
    monkeypatch.setenv("DPQ_EXACT_LIMIT", "0")
    idx3 = FlatIndex.from_arrays(cb, der, codes)
    for _ in range(3):
        d3, i3 = idx3.search(Y, 12, mode="derived", r2=200)
        assert np.array_equal(i3, outs[0][1]) and _same(d3, outs[0][0])
    assert idx3._handle().counters()["fallbacks"] > 0


@pytest.mark.parametrize("m,bits", [(4, 12), (8, 11), (3, 10), (2, 9)])
def test_direct_scan_vs_tile_scan_and_oracle(monkeypatch, m, bits):
    """The per-query direct first pass (k_key_select + k_scan_direct over the
    (g0, g1) key runs under the guard) emits exactly the tile scan's set:
    identical results with DPQ_DIRECT=0, with an item budget so small that
    part of the batch stays on the tile path (mixed batch, null-filled
    reservations), with the slack-tightened group tables off, and against
    the oracle; MPAD 4 and 8, m = 2 (no table lookups) and m = 3."""
    import torch
    from paper_1905_06900_b200 import train

    st = datagen.seed_streams(33 + m)
    centres = datagen.sift_centres(st["centres"])
    X = datagen.sift_like(st["database"], centres, 90_000)
    Y = datagen.sift_like(st["queries"], centres, 140)
    d = X.shape[1] // m * m
    X, Y = np.ascontiguousarray(X[:, :d]), np.ascontiguousarray(Y[:, :d])
    xt = torch.as_tensor(X, device="cuda")
    cb, der = train.train_pq(xt, m, bits, 4, iters=6, seed=33)  # kbar = 16
    codes = train.encode(xt, cb).cpu().numpy().astype(np.uint16)
    idx = FlatIndex.from_arrays(cb, der, codes)
    d1, i1 = idx.search(Y, 20, mode="derived", r2=150)
    b1, n1 = idx.candidate_counts(Y, 150)
    for env in ({"DPQ_DIRECT": "0"}, {"DPQ_DIRECT_ITEMS": "96"}, {"DPQ_GT_SLACK": "0"},
                {"DPQ_GRAPH": "0", "DPQ_SPECULATE": "0"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        idx2 = FlatIndex.from_arrays(cb, der, codes)
        for _ in range(2):  # (second call: graph replay)
            d2, i2 = idx2.search(Y, 20, mode="derived", r2=150)
            assert np.array_equal(i1, i2) and _same(d1, d2), env
        b2, n2 = idx2.candidate_counts(Y, 150)
        assert np.array_equal(b1, b2) and np.array_equal(n1, n2), env
        for k in env:
            monkeypatch.delenv(k)
    d0, i0 = _oracle(cb, der, codes, Y[:24], 20, 150)
    assert np.array_equal(i0, i1[:24]) and _same(d0, d1[:24])


def test_tile_skip_mode_and_fallback(monkeypatch):
    """After batches in which every query took the direct scan the tile
    kernels are not launched at all (no LUT tile loads); a later batch that
    needs them (large r2: every key admissible) is flagged by K3 and redone
    with the tile path.  Results equal the tile-only pipeline throughout."""
    import torch
    from paper_1905_06900_b200 import train

    st = datagen.seed_streams(41)
    centres = datagen.sift_centres(st["centres"])
    X = datagen.sift_like(st["database"], centres, 120_000)
    Y = datagen.sift_like(st["queries"], centres, 96)
    xt = torch.as_tensor(X, device="cuda")
    cb, der = train.train_pq(xt, 4, 12, 4, iters=6, seed=41)
    codes = train.encode(xt, cb).cpu().numpy().astype(np.uint16)
    idx = FlatIndex.from_arrays(cb, der, codes)
    monkeypatch.setenv("DPQ_DIRECT", "0")
    ref = FlatIndex.from_arrays(cb, der, codes)
    monkeypatch.delenv("DPQ_DIRECT")
    d_small, i_small = ref.search(Y, 10, mode="derived", r2=100)
    d_big, i_big = ref.search(Y, 10, mode="derived", r2=60_000)
    luts = lambda: idx._handle().counters_ex()["lut_loads"]
    deltas = []
    for _ in range(6):  # eager, capture, replay; then the skip mode (recapture, replay)
        l0 = luts()
        d, i = idx.search(Y, 10, mode="derived", r2=100)
        deltas.append(luts() - l0)
        assert np.array_equal(i, i_small) and _same(d, d_small)
    # (the sample-histogram tiles are loaded by k_scan_hist, not counted; the scan's are)
    assert deltas[-1] == 0, deltas
    l0 = luts()
    for _ in range(2):
        d, i = idx.search(Y, 10, mode="derived", r2=60_000)
        assert np.array_equal(i, i_big) and _same(d, d_big)
    assert luts() > l0  # the redo ran the tile scan
    for _ in range(4):
        d, i = idx.search(Y, 10, mode="derived", r2=100)
        assert np.array_equal(i, i_small) and _same(d, d_small)


@pytest.mark.parametrize("r2", [100, 2000])
def test_scan_side_histogram_equals_emit_list_histogram(monkeypatch, r2):
    """DPQ_SCAN_HIST=1: the direct scan counts its hits by score and K3 takes b*
    from those counts instead of reading the emit lists back (the default for
    shards of 2^24 rows or more).  Same ids, distances and refined-candidate
    counts as with DPQ_SCAN_HIST=0, batch after batch (eager, captured graph,
    tile-skip mode), and as the oracle."""
    import torch
    from paper_1905_06900_b200 import train

    st = datagen.seed_streams(43)
    centres = datagen.sift_centres(st["centres"])
    X = datagen.sift_like(st["database"], centres, 150_000)
    Y = datagen.sift_like(st["queries"], centres, 64)
    xt = torch.as_tensor(X, device="cuda")
    cb, der = train.train_pq(xt, 4, 12, 4, iters=6, seed=43)
    codes = train.encode(xt, cb).cpu().numpy().astype(np.uint16)
    monkeypatch.setenv("DPQ_SCAN_HIST", "0")
    off = FlatIndex.from_arrays(cb, der, codes)
    monkeypatch.setenv("DPQ_SCAN_HIST", "1")
    on = FlatIndex.from_arrays(cb, der, codes)
    d0, i0 = O.flat_search(cb, der, codes, Y[:8], 10, "derived", r2)
    for _ in range(5):
        refined = []
        res = []
        for idx in (off, on):
            c0 = idx._handle().counters_ex()["refined"]
            res.append(idx.search(Y, 10, mode="derived", r2=r2))
            refined.append(idx._handle().counters_ex()["refined"] - c0)
        assert np.array_equal(res[0][1], res[1][1]) and _same(res[0][0], res[1][0])
        assert refined[0] == refined[1], refined
        assert np.array_equal(res[1][1][:8], i0) and _same(res[1][0][:8], d0)


def test_deferred_finiteness_check_raises_like_check_array():
    """Once the device handle exists the finiteness scan of check_array rides
    on libdpq's staging copy (dpq_set_check_finite): NaN / infinity still
    raise sklearn's ValueError, before any other argument error, in every
    batch of a multi-batch call, and valid calls keep working afterwards."""
    cb, der, codes, Y = _sift_setup(20_000, 40, seed=23)
    idx = FlatIndex.from_arrays(cb, der, codes)
    d0, i0 = idx.search(Y, 5, mode="derived", r2=100)  # creates the handle (eager check on this call)
    bad = Y.copy()
    bad[7, 3] = np.inf
    with pytest.raises(ValueError, match="infinity"):
        idx.search(bad, 5, mode="derived", r2=100)
    with pytest.raises(ValueError, match="infinity"):
        idx.search(bad, 5)  # conventional
    bad[30, 0] = np.nan
    with pytest.raises(ValueError, match="NaN"):
        idx.search(bad, 5, mode="derived", r2=100)
    with pytest.raises(ValueError, match="NaN"):  # the reference checks the array before its other arguments
        idx.search(bad, 5, mode="blended")
    with pytest.raises(ValueError, match="unknown mode"):
        idx.search(Y, 5, mode="blended")
    idx._handle().set_batch(16)  # the bad row sits in the third batch
    with pytest.raises(ValueError, match="NaN"):
        idx.search(bad, 5, mode="derived", r2=100)
    idx._handle().set_batch(1024)
    d1, i1 = idx.search(Y, 5, mode="derived", r2=100)
    assert np.array_equal(i0, i1) and _same(d0, d1)


def test_device_buffer_api_single_and_multi_batch():
    """dpq_flat_search_derived_dev (queries and results in device memory): a
    call that is one batch has the refine write straight into the caller's
    buffers (graph keyed on them), a longer call goes through the workspace;
    both equal the host API, also when the output buffers change between
    calls."""
    import torch
    from paper_1905_06900_b200 import _lib

    cb, der, codes, Y = _sift_setup(60_000, 100, seed=29)
    idx = FlatIndex.from_arrays(cb, der, codes)
    d0, i0 = idx.search(Y, 7, mode="derived", r2=120)
    h, L = idx._handle(), _lib.lib()
    q = torch.as_tensor(Y, device="cuda")
    for batch in (1024, 32):  # one batch / four batches
        h.set_batch(batch)
        for rep in range(4):  # eager, capture, replay, new output buffers
            od = torch.full((100, 7), -1.0, dtype=torch.float64, device="cuda")
            oi = torch.full((100, 7), -7, dtype=torch.int64, device="cuda")
            _lib.check(L.dpq_flat_search_derived_dev(h.raw, _lib.ptr(q), 100, 7, 120, _lib.ptr(od), _lib.ptr(oi)))
            torch.cuda.synchronize()
            assert np.array_equal(oi.cpu().numpy(), i0) and _same(od.cpu().numpy(), d0), (batch, rep)
    h.set_batch(1024)
