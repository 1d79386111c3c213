"""Tensor-core full tables (dpq_tctab.cu, north_star (i)): the tcgen05
3xTF32 approximation of compute_tables (search.py:28-48) stays inside its
stated error bound and within the north_star tolerance (1e-4 relative), and
the derived search that consumes it (exact re-rank of the margin set) is
still bit-identical to the reference."""

import numpy as np
import pytest

from conftest import FLAT_CASES, load_golden
from oracle import derived_search as O
from paper_1905_06900_b200.flat import FlatIndex

pytestmark = pytest.mark.gpu


def _same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))


def _check_tables(idx, Y, rel_tol=1e-4):
    approx, eps = idx.tc_tables(Y)
    exact = idx.full_tables(Y)  # numpy's bits (CUDA-core kernel, bitwise per test_gpu_flat)
    err = np.abs(approx.astype(np.float64) - exact.astype(np.float64))
    assert np.all(err <= eps[:, :, None]), float((err / eps[:, :, None]).max())
    # north_star: LUT values within 1e-4 relative (of the table's scale per query and subspace)
    scale = np.maximum(np.abs(exact).max(axis=2, keepdims=True), 1e-30)
    assert float((err / scale).max()) <= rel_tol
    return float((err / eps[:, :, None]).max())


@pytest.mark.parametrize("name", FLAT_CASES)
def test_tc_tables_within_bound_goldens(name):
    g = load_golden(name)
    idx = FlatIndex.from_arrays(g["codebooks"], g["derived"], g["codes"], rotation=g.get("rotation"))
    _check_tables(idx, g["queries"])


def test_tc_tables_config1_shape(c1_golden):
    g = c1_golden
    idx = FlatIndex.from_arrays(g["codebooks"], g["derived"], g["codes"])
    _check_tables(idx, g["queries"][:24])


@pytest.mark.parametrize("name", FLAT_CASES)
@pytest.mark.parametrize("scale", ["1", "1000"])
def test_derived_search_tc_bitwise_vs_reference(name, scale, monkeypatch):
    """Forced tensor-core tables (and a 1000x looser bound: far more exact
    re-ranks) give the reference's bits."""
    monkeypatch.setenv("DPQ_TC_TABLES", "1")
    monkeypatch.setenv("DPQ_TC_EPS_SCALE", scale)
    g = load_golden(name)
    m = g["meta"]
    idx = FlatIndex.from_arrays(g["codebooks"], g["derived"], g["codes"], rotation=g.get("rotation"))
    d, i = idx.search(g["queries"], m["r"], mode="derived", r2=m["r2"])
    assert np.array_equal(i, g["exp_derived_i"])
    assert _same(d, g["exp_derived_d"])
    c = idx._handle().counters_ex()
    assert c["exact_reranked"] > 0


def test_derived_search_tc_config1_shape(c1_golden, monkeypatch):
    monkeypatch.setenv("DPQ_TC_TABLES", "1")
    g = c1_golden
    m = g["meta"]
    d, i = FlatIndex.from_arrays(g["codebooks"], g["derived"], g["codes"]).search(g["queries"], m["r"],
                                                                               mode="derived", r2=m["r2"])
    assert np.array_equal(i, g["exp_derived_i"])
    assert _same(d, g["exp_derived_d"])


def _gist_model(seed, m=8, k=65536, kbar=256, dsub=120, n=20000, nq=12):
    """8 x 65536 x 120 (BASELINE configs[4] shape): codebooks from seeded
    GIST-like points, derived codebooks = group means, random codes."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0, 1, size=(64, dsub))
    cb = np.clip(centres[rng.integers(64, size=(m, k))] + rng.normal(0, 0.05, size=(m, k, dsub)), 0, 1)
    cb = cb.astype(np.float32)
    der = np.stack([cb[j].reshape(k // kbar, kbar, dsub).astype(np.float64).mean(axis=0) for j in range(m)])
    der = der.astype(np.float32)
    codes = rng.integers(0, k, size=(n, m)).astype(np.uint16)
    # database-like codes: rows near a few centroids of each subspace, so candidates cluster
    Y = np.clip(centres[rng.integers(64, size=(nq, m))].reshape(nq, m * dsub)
                + rng.normal(0, 0.05, size=(nq, m * dsub)), 0, 1).astype(np.float32)
    return cb, der, codes, Y


def test_tc_tables_gist_8x65536x120(monkeypatch):
    cb, der, codes, Y = _gist_model(5)
    idx = FlatIndex.from_arrays(cb, der, codes)
    ratio = _check_tables(idx, Y[:6])
    assert ratio < 1.0


def test_derived_search_tc_gist_vs_oracle(monkeypatch):
    """configs[4] shape (m = 8, dsub = 120) through the default path (tensor-
    core tables for dsub >= 64): bit-identical to the oracle."""
    cb, der, codes, Y = _gist_model(6, nq=6)
    r, r2 = 50, 600
    idx = FlatIndex.from_arrays(cb, der, codes)
    d, i = idx.search(Y, r, mode="derived", r2=r2)
    d0, i0 = O.flat_search(cb, der, codes, Y, r, "derived", r2)
    assert np.array_equal(i, i0)
    assert _same(d, d0)
    c = idx._handle().counters_ex()
    assert c["exact_reranked"] >= r * Y.shape[0]
    monkeypatch.setenv("DPQ_TC_TABLES", "0")  # the lazy exact builder gives the same bits
    d2, i2 = FlatIndex.from_arrays(cb, der, codes).search(Y, r, mode="derived", r2=r2)
    assert np.array_equal(i2, i0) and _same(d2, d0)
