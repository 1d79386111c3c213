"""Unit seams of the drop-in boundary: the GPU twins of
adc_low_batch (twopass.py:99-106) and of the candidate list the refine walk
scores (scan_derived + CappedBuckets + refine, twopass.py:171-217, 276-302),
checked bit-exactly against the reference's golden outputs and the oracle.
"""

import numpy as np
import pytest

from conftest import FLAT_CASES, load_golden
from oracle import derived_search as O
from paper_1905_06900_b200.flat import FlatIndex

pytestmark = pytest.mark.gpu


def _index(g, codebooks=None):
    return FlatIndex.from_arrays(g["codebooks"] if codebooks is None else codebooks, g["derived"], g["codes"],
                                 rotation=g.get("rotation"))


def _oracle_scores(g, qi):
    bbar = int(g["derived"].shape[1]).bit_length() - 1
    qt = O.Quantized(g["exp_q"][qi], float(g["exp_qmin"][qi]), float(g["exp_qmax"][qi]), bbar)
    return O.low_scores(g["codes"], qt)


@pytest.mark.parametrize("name", FLAT_CASES)
def test_low_scores_bitwise(name):
    g = load_golden(name)
    got = _index(g).low_scores(g["queries"], g["meta"]["r2"])
    assert got.shape == (g["queries"].shape[0], g["codes"].shape[0])
    for qi in range(g["queries"].shape[0]):
        assert np.array_equal(got[qi], _oracle_scores(g, qi)), qi


@pytest.mark.parametrize("name", FLAT_CASES)
def test_candidate_ids_bucket_walk(name):
    g = load_golden(name)
    r2 = g["meta"]["r2"]
    cands = _index(g).candidate_ids(g["queries"], r2)
    n = g["codes"].shape[0]
    for qi, (ids, sc) in enumerate(cands):
        s = _oracle_scores(g, qi)
        want = O.bucket_walk(s, np.arange(n, dtype=np.int64), r2)
        assert np.array_equal(ids, want), qi
        assert np.array_equal(sc, s[want])
        assert len(ids) == g["exp_ncand"][qi]  # the reference's own walk count
        if len(ids):
            assert int(sc.max()) == int(g["exp_bwalk"][qi])  # the last bucket the walk took


def test_candidate_ids_config1_shape(c1_golden):
    """PQ 4x16/8 over N = 100k (rows sorted by (g0, g1) inside the index):
    ids come back in the caller's row numbering, in walk order."""
    g = c1_golden
    idx = _index(g, g["codebooks"])
    Y = g["queries"][:8]
    r2 = g["meta"]["r2"]
    small, q, qmin, qmax = idx.quantized_tables(Y, r2)
    scores = idx.low_scores(Y, r2)
    cands = idx.candidate_ids(Y, r2)
    bstar, ncand = idx.candidate_counts(Y, r2)
    n = g["codes"].shape[0]
    for qi in range(Y.shape[0]):
        s = O.low_scores(g["codes"], O.Quantized(q[qi], float(qmin[qi]), float(qmax[qi]), 8))
        assert np.array_equal(scores[qi], s)
        want = O.bucket_walk(s, np.arange(n, dtype=np.int64), r2)
        ids, sc = cands[qi]
        assert np.array_equal(ids, want)
        assert len(ids) == ncand[qi] and int(sc.max()) == bstar[qi]
