"""Host-side behaviour of the drop-in mirrors that does not need a GPU:
argument validation order, exception types and messages (flat.py:70-96,
twopass.py:330-331, ivf.py:125-140 of the reference), empty batches, the
oracle-free merge helper, and that searches fail loudly without a device."""

import numpy as np
import pytest
from sklearn.exceptions import NotFittedError

from conftest import load_golden
from paper_1905_06900_b200 import ArrayQuantizer, FlatIndex, IVFIndex
from paper_1905_06900_b200 import _lib


@pytest.fixture()
def flat():
    g = load_golden("pq_blobs")
    return FlatIndex.from_arrays(g["codebooks"], g["derived"], g["codes"]), g


def test_not_fitted_raises_sklearn_error():
    q = ArrayQuantizer(np.zeros((2, 4, 2), np.float32), np.zeros((2, 2, 2), np.float32))
    with pytest.raises(NotFittedError):
        FlatIndex(q).search(np.zeros((1, 4), np.float32), 1)
    with pytest.raises(NotFittedError):
        IVFIndex(q).search(np.zeros((1, 4), np.float32), 1)


def test_validation_before_device(flat):
    idx, g = flat
    Y = g["queries"][:2]
    with pytest.raises(ValueError, match="mode"):
        idx.search(Y, 5, mode="hybrid")
    with pytest.raises(ValueError, match="r2"):
        idx.search(Y, 5, mode="derived")
    with pytest.raises(ValueError, match="must not exceed"):
        idx.search(Y, 11, mode="derived", r2=10)
    with pytest.raises(ValueError, match="dimension"):
        idx.search(np.zeros((2, 3), np.float32), 5)  # compute_tables (search.py:42-43)
    with pytest.raises(ValueError, match="result size"):
        idx.search(Y, 0)


def test_empty_batch_rejected_like_reference(flat):
    # the reference's check_array (flat.py:71) rejects a 0-row query array
    idx, g = flat
    with pytest.raises(ValueError, match="0 sample"):
        idx.search(np.zeros((0, g["queries"].shape[1]), np.float32), 7, mode="derived", r2=20)


def test_empty_database_derived_raises(flat):
    _, g = flat
    idx = FlatIndex.from_arrays(g["codebooks"], g["derived"], g["codes"][:0])
    with pytest.raises(ValueError, match="at least one code"):
        idx.search(g["queries"][:1], 1, mode="derived", r2=5)


def test_ivf_validation(flat):
    g = load_golden("ivf_blobs")
    idx = IVFIndex.from_arrays(g["codebooks"], g["derived"], g["centers"], g["offsets"], g["sorted_codes"],
                               g["sorted_ids"], cell_of=g["cell_of"])
    Y = g["queries"][:1]
    with pytest.raises(ValueError, match="mode"):
        idx.search(Y, 5, mode="blended")
    with pytest.raises(ValueError, match="r2"):
        idx.search(Y, 5, mode="derived")
    with pytest.raises(ValueError):
        idx.search(Y, 5, mode="derived", r2=3)
    with pytest.raises(ValueError, match="ma must be"):
        idx.probe(Y[0], 0)
    with pytest.raises(ValueError, match="ma must be"):
        idx.search(Y, 5, ma=17)
    # row_of_ / cell_of_ reconstruction in from_arrays
    assert np.array_equal(idx.sorted_ids_[idx.row_of_], np.arange(idx.n_))
    assert np.array_equal(idx.cell_of_, g["cell_of"])


def test_search_without_device_fails_loudly(flat):
    if _lib.device_count() > 0:
        pytest.skip("a device is present")
    idx, g = flat
    with pytest.raises(RuntimeError, match="not available"):
        idx.search(g["queries"][:1], 5, mode="derived", r2=50)


def test_array_quantizer_rotate_matches_reference_semantics():
    rng = np.random.default_rng(0)
    R = np.linalg.qr(rng.normal(size=(8, 8)))[0].astype(np.float32)
    q = ArrayQuantizer(np.zeros((2, 4, 4), np.float32), np.zeros((2, 2, 4), np.float32), rotation=R)
    X = rng.normal(size=(3, 8)).astype(np.float32)
    assert np.array_equal(q.rotate(X), (X @ R).astype(np.float32))
    assert q.rotate(X).dtype == np.float32


def test_non_finite_queries_rejected_like_check_array(flat):
    """The native finiteness fast path raises sklearn's own messages, NaN
    before infinity, for flat and ivf searches (flat.py:71, ivf.py:125)."""
    idx, g = flat
    Y = np.array(g["queries"][:3], dtype=np.float32)
    Y[1, 2] = np.inf
    with pytest.raises(ValueError, match="infinity"):
        idx.search(Y, 5, mode="derived", r2=20)
    Y[2, 0] = np.nan
    with pytest.raises(ValueError, match="NaN"):
        idx.search(Y, 5)
    assert _lib.lib().dpq_all_finite(Y[:1].ctypes.data, Y[:1].size) == 0
    # non-float32 / non-contiguous input still goes through check_array
    idx2 = FlatIndex.from_arrays(g["codebooks"], g["derived"], g["codes"])
    with pytest.raises(ValueError, match="NaN"):
        idx2.search(np.asfortranarray(Y.astype(np.float64)), 5)


def test_encoder_without_device_fails_loudly():
    """The tensor-core encoder has no CPU fallback either."""
    if _lib.device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(RuntimeError, match="not available"):
        _lib.Encoder(np.zeros((1, 16, 8), np.float32))


def test_train_make_encoder_kinds():
    from paper_1905_06900_b200 import train

    with pytest.raises(ValueError, match="unknown encoder"):
        train.make_encoder(np.zeros((1, 4, 2), np.float32), kind="nope")


def test_finiteness_scan_parallel_path():
    """dpq_all_finite on > 256 KB (the multi-threaded branch): finite, NaN
    and inf anywhere, NaN winning over inf (check_array's order)."""
    L = _lib.lib()
    x = np.random.default_rng(1).normal(size=(4096, 128)).astype(np.float32)
    assert L.dpq_all_finite(_lib.ptr(x), x.size) == 0
    x[4000, 7] = np.inf
    assert L.dpq_all_finite(_lib.ptr(x), x.size) == 2
    x[10, 0] = np.nan
    assert L.dpq_all_finite(_lib.ptr(x), x.size) == 1
