"""Pin the CPU oracle against outputs of the reference itself.

tests/golden/*.npz were produced by the unmodified derivedpq package
(tests/golden/make_golden.py).  Every comparison here is exact: the oracle
must reproduce the reference's float bits, not approximate them, because it
is the checker the CUDA path is held to on the GPU box.
"""

import numpy as np
import pytest

from conftest import FLAT_CASES, IVF_CASES, load_golden
from oracle import derived_search as O


def _rot(g):
    return O.make_rotate(g.get("rotation"))


@pytest.mark.parametrize("name", FLAT_CASES)
def test_small_tables_and_quantization_bitwise(name):
    g = load_golden(name)
    rot, r2 = _rot(g), g["meta"]["r2"]
    for qi, y in enumerate(g["queries"]):
        yr = rot(y.reshape(1, -1)).reshape(-1)
        small = O.lookup_tables(yr, g["derived"])
        qt = O.quantize_small(small, g["codes"][: min(r2, len(g["codes"]))], r2)
        assert np.array_equal(small.view(np.uint32), g["exp_small"][qi].view(np.uint32))
        assert np.array_equal(qt.q, g["exp_q"][qi])
        assert qt.qmin == g["exp_qmin"][qi] and qt.qmax == g["exp_qmax"][qi]


@pytest.mark.parametrize("name", FLAT_CASES)
def test_candidate_walk_matches_reference(name):
    g = load_golden(name)
    rot, r2 = _rot(g), g["meta"]["r2"]
    for qi, y in enumerate(g["queries"]):
        _, _, info = O.derived_one(g["codebooks"], g["derived"], rot, g["codes"], y, 1, r2)
        assert info["ncand"] == g["exp_ncand"][qi]
        # closed form of the walk (SURVEY Appendix A rule 8)
        bstar = O.closed_form_bstar(info["scores"], r2)
        s = info["scores"]
        assert int(((s <= bstar) & (s < 255)).sum()) == g["exp_ncand"][qi]


@pytest.mark.parametrize("name", FLAT_CASES)
def test_flat_derived_results_bitwise(name):
    g = load_golden(name)
    m = g["meta"]
    d, i = O.flat_search(g["codebooks"], g["derived"], g["codes"], g["queries"], m["r"], "derived",
                         m["r2"], rotation=g.get("rotation"))
    assert np.array_equal(i, g["exp_derived_i"])
    assert np.array_equal(d.view(np.uint64), g["exp_derived_d"].view(np.uint64))


@pytest.mark.parametrize("name", FLAT_CASES)
def test_flat_conventional_and_full_budget(name):
    g = load_golden(name)
    m = g["meta"]
    if "exp_conv_i" in g:
        d, i = O.flat_search(g["codebooks"], g["derived"], g["codes"], g["queries"], m["r"],
                             rotation=g.get("rotation"))
        assert np.array_equal(i, g["exp_conv_i"])
        assert np.array_equal(d, g["exp_conv_d"])
    if "exp_full_i" in g:
        r = g["exp_full_i"].shape[1]
        d, i = O.flat_search(g["codebooks"], g["derived"], g["codes"], g["queries"][:4], r, "derived",
                             len(g["codes"]), capped=False, rotation=g.get("rotation"))
        assert np.array_equal(i, g["exp_full_i"])
        assert np.array_equal(d, g["exp_full_d"])


def _ivf(g):
    n = g["sorted_ids"].shape[0]
    row_of = np.empty(n, np.int64)
    row_of[g["sorted_ids"]] = np.arange(n)
    kbar = g["derived"].shape[1]
    return {"centers": g["centers"], "offsets": g["offsets"], "sorted_codes": g["sorted_codes"],
            "sorted_ids": g["sorted_ids"], "cell_of": g["cell_of"], "row_of": row_of,
            "codebooks": g["codebooks"], "derived": g["derived"], "bbar": int(kbar).bit_length() - 1,
            "rotate": O.make_rotate(g.get("rotation"))}


@pytest.mark.parametrize("name", IVF_CASES)
def test_ivf_results_bitwise(name):
    g = load_golden(name)
    m = g["meta"]
    ivf = _ivf(g)
    for qi, y in enumerate(g["queries"]):
        cells, _ = O.ivf_probe(g["centers"], y, m["ma"])
        assert np.array_equal(cells, g["exp_cells"][qi])
    d, i = O.ivf_search(ivf, g["queries"], m["r"], m["ma"], "derived", m["r2"])
    assert np.array_equal(i, g["exp_derived_i"])
    assert np.array_equal(d, g["exp_derived_d"])
    d, i = O.ivf_search(ivf, g["queries"], m["r"], m["ma"])
    assert np.array_equal(i, g["exp_conv_i"])
    assert np.array_equal(d, g["exp_conv_d"])
    d, i = O.ivf_search(ivf, g["queries"][:4], 8, m["n_cells"], "derived", m["n"], capped=False)
    assert np.array_equal(i, g["exp_full_i"])
    assert np.array_equal(d, g["exp_full_d"])


def test_config1_shape_oracle(c1_golden):
    g = c1_golden
    m = g["meta"]
    sel = slice(0, 12)  # the oracle costs ~0.3 s/query at this size
    d, i = O.flat_search(g["codebooks"], g["derived"], g["codes"], g["queries"][sel], m["r"], "derived",
                         m["r2"])
    assert np.array_equal(i, g["exp_derived_i"][sel])
    assert np.array_equal(d, g["exp_derived_d"][sel])


def test_bucket_walk_equals_closed_form_random():
    """The refine walk's candidate count equals |{s <= b*}| (Appendix A
    rule 8) for random score multisets, capped or not."""
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = int(rng.integers(1, 400))
        r2 = int(rng.integers(1, 80))
        hi = int(rng.integers(1, 257))
        scores = rng.integers(0, hi, size=n).astype(np.uint8)
        ids = rng.permutation(n)
        for capped in (True, False):
            cand = O.bucket_walk(scores, ids, r2, capped)
            b = O.closed_form_bstar(scores, r2)
            expect = set(ids[(scores <= b) & (scores < 255)].tolist())
            assert set(cand.tolist()) == expect
