"""Parity of the CUDA IVF path with the reference (golden fixtures) and the
CPU oracle on seeded inputs.  Bar: bit-exact ids and f64 distances."""

import numpy as np
import pytest

from conftest import IVF_CASES, load_golden
from oracle import derived_search as O
from paper_1905_06900_b200 import datagen
from paper_1905_06900_b200.ivf import IVFIndex

pytestmark = pytest.mark.gpu


def _same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))


def _index(g):
    return IVFIndex.from_arrays(g["codebooks"], g["derived"], g["centers"], g["offsets"], g["sorted_codes"],
                                g["sorted_ids"], cell_of=g["cell_of"], rotation=g.get("rotation"))


def _oracle_ivf(idx):
    kbar = idx.quantizer.derived_codebooks_.shape[1]
    return {"centers": idx.centers_, "offsets": idx.offsets_, "sorted_codes": idx.sorted_codes_,
            "sorted_ids": idx.sorted_ids_, "cell_of": idx.cell_of_, "row_of": idx.row_of_,
            "codebooks": idx.quantizer.codebooks_, "derived": idx.quantizer.derived_codebooks_,
            "bbar": int(kbar).bit_length() - 1, "rotate": O.make_rotate(idx.quantizer.rotation_)}


@pytest.mark.parametrize("name", IVF_CASES)
def test_probe_matches_reference(name):
    g = load_golden(name)
    idx = _index(g)
    ma = g["meta"]["ma"]
    for qi, y in enumerate(g["queries"]):
        cells, res = idx.probe(y, ma)
        assert np.array_equal(cells, g["exp_cells"][qi])
        assert np.array_equal(res, y[None, :] - g["centers"][cells])


@pytest.mark.parametrize("name", IVF_CASES)
def test_ivf_derived_bitwise_vs_reference(name):
    g = load_golden(name)
    m = g["meta"]
    d, i = _index(g).search(g["queries"], m["r"], ma=m["ma"], mode="derived", r2=m["r2"])
    assert np.array_equal(i, g["exp_derived_i"])
    assert _same(d, g["exp_derived_d"])


@pytest.mark.parametrize("name", IVF_CASES)
def test_ivf_conventional_and_full_budget_vs_reference(name):
    g = load_golden(name)
    m = g["meta"]
    idx = _index(g)
    d, i = idx.search(g["queries"], m["r"], ma=m["ma"])
    assert np.array_equal(i, g["exp_conv_i"]) and _same(d, g["exp_conv_d"])
    d, i = idx.search(g["queries"][:4], 8, ma=m["n_cells"], mode="derived", r2=m["n"], capped=False)
    assert np.array_equal(i, g["exp_full_i"]) and _same(d, g["exp_full_d"])


def _random_ivf(seed, n, K, m=4, k=256, kbar=16, dsub=4, empty=0):
    rng = np.random.default_rng(seed)
    d = m * dsub
    centers = rng.normal(size=(K, d)).astype(np.float32) * 4
    cb = rng.normal(size=(m, k, dsub)).astype(np.float32)
    der = np.stack([np.stack([cb[j][np.arange(k) % kbar == gg].mean(axis=0) for gg in range(kbar)])
                    for j in range(m)]).astype(np.float32)
    cell_of = rng.integers(0, K - empty, size=n)
    order = np.argsort(cell_of, kind="stable").astype(np.int64)
    codes = rng.integers(0, k, size=(n, m)).astype(np.uint8 if k <= 256 else np.uint16)
    counts = np.bincount(cell_of, minlength=K)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    idx = IVFIndex.from_arrays(cb, der, centers, offsets, codes[order], order, cell_of=cell_of)
    Y = (centers[rng.integers(0, K, size=17)] + rng.normal(size=(17, d))).astype(np.float32)
    return idx, Y


@pytest.mark.parametrize("seed,n,K,ma,r,r2,empty", [
    (1, 4000, 16, 4, 10, 300, 0),
    (2, 3000, 32, 8, 20, 500, 5),      # empty lists among the probed ones
    (3, 2500, 1, 1, 10, 100, 0),       # K = 1
    (4, 2000, 8, 8, 50, 2000, 0),      # probe everything, full budget
    (5, 500, 64, 3, 40, 60, 30),       # many empty / tiny lists, padding
])
def test_random_ivf_vs_oracle(seed, n, K, ma, r, r2, empty):
    idx, Y = _random_ivf(seed, n, K, empty=empty)
    ivf = _oracle_ivf(idx)
    d0, i0 = O.ivf_search(ivf, Y, r, ma, "derived", r2)
    d1, i1 = idx.search(Y, r, ma=ma, mode="derived", r2=r2)
    assert np.array_equal(i0, i1)
    assert _same(d0, d1)
    d0, i0 = O.ivf_search(ivf, Y, r, ma)
    d1, i1 = idx.search(Y, r, ma=ma)
    assert np.array_equal(i0, i1) and _same(d0, d1)


@pytest.mark.parametrize("seed", [21, 22, 23])
@pytest.mark.parametrize("n,K,ma,r,r2,empty", [(4000, 16, 4, 10, 300, 0), (3000, 32, 8, 20, 500, 5),
                                               (500, 64, 3, 40, 60, 30), (8000, 128, 16, 50, 800, 40)])
def test_random_ivf_more_seeds(seed, n, K, ma, r, r2, empty):
    """More seeds, plus single-query searches against the batched ones."""
    idx, Y = _random_ivf(seed * 31 + K, n, K, empty=empty)
    ivf = _oracle_ivf(idx)
    d0, i0 = O.ivf_search(ivf, Y, r, ma, "derived", r2)
    d1, i1 = idx.search(Y, r, ma=ma, mode="derived", r2=r2)
    assert np.array_equal(i0, i1) and _same(d0, d1)
    for qi in range(3):
        d2, i2 = idx.search(Y[qi:qi + 1], r, ma=ma, mode="derived", r2=r2)
        assert np.array_equal(i2[0], i0[qi]) and _same(d2[0], d0[qi])


@pytest.mark.parametrize("dsub,kbar", [(8, 16), (16, 256), (32, 64)])
def test_many_slot_tables_vs_oracle(dsub, kbar, monkeypatch):
    """The many-slot K1 (8 slots per CTA, paired-FP32 entries) that IVF
    batches with >= 8192 live slots use, forced on small batches."""
    monkeypatch.setenv("DPQ_MS_MIN", "1")
    idx, Y = _random_ivf(11 + dsub, 6000, 24, k=1024, kbar=kbar, dsub=dsub, empty=3)
    ivf = _oracle_ivf(idx)
    d0, i0 = O.ivf_search(ivf, Y, 30, 6, "derived", 400)
    d1, i1 = idx.search(Y, 30, ma=6, mode="derived", r2=400)
    assert np.array_equal(i0, i1) and _same(d0, d1)


def test_ivf_sampled_guard_vs_oracle(monkeypatch):
    """Long lists: the per-query guard comes from strided list samples; a tiny
    sample forces exact redos."""
    monkeypatch.setenv("DPQ_EXACT_LIMIT", "0")
    monkeypatch.setenv("DPQ_GUARD_SAMPLE", "64")
    idx, Y = _random_ivf(9, 60000, 8, k=1024, kbar=64)
    ivf = _oracle_ivf(idx)
    d0, i0 = O.ivf_search(ivf, Y[:6], 25, 3, "derived", 800)
    d1, i1 = idx.search(Y[:6], 25, ma=3, mode="derived", r2=800)
    assert np.array_equal(i0, i1) and _same(d0, d1)


def test_ivf_errors_and_timings():
    g = load_golden("ivf_blobs")
    idx = _index(g)
    with pytest.raises(ValueError, match="r2"):
        idx.search(g["queries"][:1], 5, mode="derived")
    with pytest.raises(ValueError):
        idx.search(g["queries"][:1], 5, mode="derived", r2=3)
    with pytest.raises(ValueError, match="mode"):
        idx.search(g["queries"][:1], 5, mode="blended")
    with pytest.raises(ValueError):
        idx.probe(g["queries"][0], 0)
    with pytest.raises(ValueError):
        idx.probe(g["queries"][0], 17)
    _, _, t = idx.search(g["queries"][:4], 5, ma=4, return_timings=True)
    assert set(t) == {"index_us", "tables_us", "scan_us", "refine_us"}
    assert np.all(t["refine_us"] == 0.0)
    dists, ids = idx.search(g["queries"][:1], 6000, ma=1)
    n_found = int((ids[0] >= 0).sum())
    assert 0 < n_found < 6000 and np.all(np.isinf(dists[0, n_found:]))


# ---- tensor-core probe (k_probe_select_tc): same cells, same order, as the f64 probe ----

def _probe_all(idx, Y, ma):
    return idx._probe_cells(np.ascontiguousarray(Y, dtype=np.float32), ma)


@pytest.mark.parametrize("name", IVF_CASES)
def test_tc_probe_forced_matches_reference(monkeypatch, name):
    g = load_golden(name)
    K = g["centers"].shape[0]
    if K % 4:
        pytest.skip("tensor-core tables need 4 | K")
    monkeypatch.setenv("DPQ_PROBE_TC", "2")
    idx = _index(g)
    m = g["meta"]
    cells = _probe_all(idx, g["queries"], m["ma"])
    assert np.array_equal(cells, g["exp_cells"])
    d, i = idx.search(g["queries"], m["r"], ma=m["ma"], mode="derived", r2=m["r2"])
    assert np.array_equal(i, g["exp_derived_i"]) and _same(d, g["exp_derived_d"])


@pytest.mark.parametrize("K,d,ma", [(2048, 128, 64), (8192, 128, 64), (1024, 96, 7), (4096, 128, 1)])
def test_tc_probe_equals_f64_probe(monkeypatch, K, d, ma):
    rng = np.random.default_rng(K + d)
    centers = rng.uniform(0, 64, size=(K, d)).astype(np.float32)
    centers[5] = centers[9]          # exact distance ties: the lower cell first
    centers[K - 1] = centers[3]
    Y = np.concatenate([rng.uniform(0, 64, size=(200, d)), centers[[3, 5, 100]] + 0.0]).astype(np.float32)
    m, dsub = 2, d // 2
    cb = rng.normal(size=(m, 256, dsub)).astype(np.float32)
    der = cb[:, :16].copy()
    n = 4 * K
    codes = rng.integers(0, 256, size=(n, m)).astype(np.uint8)
    cell_of = rng.integers(0, K, size=n)
    order = np.argsort(cell_of, kind="stable")
    offsets = np.concatenate([[0], np.cumsum(np.bincount(cell_of, minlength=K))]).astype(np.int64)
    args = (cb, der, centers, offsets, codes[order], order.astype(np.int64))
    monkeypatch.setenv("DPQ_PROBE_TC", "0")
    ref = _probe_all(IVFIndex.from_arrays(*args, cell_of=cell_of), Y, ma)
    monkeypatch.setenv("DPQ_PROBE_TC", "2")
    idx = IVFIndex.from_arrays(*args, cell_of=cell_of)
    got = _probe_all(idx, Y, ma)
    assert np.array_equal(got, ref)
    # and the reference's own rule (ivf.py:117-120): f64 distances, ascending, lower id on ties
    for q in (0, 7, Y.shape[0] - 1):
        diff = centers.astype(np.float64) - Y[q].astype(np.float64)
        d2 = np.einsum("kd,kd->k", diff, diff)
        exp = np.lexsort((np.arange(K), d2))[:ma]
        assert np.array_equal(got[q], exp)
    assert idx._handle().counters_ex()["probe_exact"] >= ma * Y.shape[0]


@pytest.mark.parametrize("sample,exact_limit", [("64", "0"), (None, None)])
def test_device_plan_equals_host_plan(monkeypatch, sample, exact_limit):
    """The device-built IVF plan (stable radix sort of probes by cell) and the
    host plan give the same results, sampled guards and exact ones."""
    rng = np.random.default_rng(11)
    K, d, m = 256, 32, 4
    centers = rng.uniform(0, 64, size=(K, d)).astype(np.float32)
    cb = rng.normal(size=(m, 256, d // m)).astype(np.float32)
    der = cb[:, :16].copy()
    n = 60_000
    cell_of = rng.integers(0, K, size=n)
    cell_of[cell_of % 7 == 3] = 5            # a few long lists, several empty cells
    order = np.argsort(cell_of, kind="stable")
    offsets = np.concatenate([[0], np.cumsum(np.bincount(cell_of, minlength=K))]).astype(np.int64)
    codes = rng.integers(0, 256, size=(n, m)).astype(np.uint8)
    args = (cb, der, centers, offsets, codes[order], order.astype(np.int64))
    Y = rng.uniform(0, 64, size=(300, d)).astype(np.float32)
    if sample:
        monkeypatch.setenv("DPQ_GUARD_SAMPLE", sample)
        monkeypatch.setenv("DPQ_EXACT_LIMIT", exact_limit)
    out = {}
    for dev in ("0", "1"):
        monkeypatch.setenv("DPQ_IVF_DEVPLAN", dev)
        idx = IVFIndex.from_arrays(*args, cell_of=cell_of)
        out[dev] = idx.search(Y, 10, ma=16, mode="derived", r2=200)
    assert np.array_equal(out["0"][1], out["1"][1]) and _same(out["0"][0], out["1"][0])
    d0, i0 = O.ivf_search(_oracle_ivf(idx), Y[:3], 10, 16, "derived", 200)
    assert np.array_equal(i0, out["1"][1][:3]) and _same(d0, out["1"][0][:3])
