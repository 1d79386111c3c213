"""quantizer.rotate in the reference's call shapes through numpy's own BLAS
(dpq_rotate_rows, host only): bit-identical to calling rotate per query —
(1, d) rows for the flat search (twopass.py:334), (ma, d) residual blocks for
IVF (ivf.py:202) — SURVEY Appendix A rule 11."""

import numpy as np
import pytest

from conftest import load_golden
from paper_1905_06900_b200 import _lib
from paper_1905_06900_b200.flat import ArrayQuantizer, rotated_queries


def _quantizer(d=128, seed=1):
    rng = np.random.default_rng(seed)
    R = np.linalg.qr(rng.normal(size=(d, d)))[0].astype(np.float32)
    return ArrayQuantizer(np.zeros((4, 16, d // 4), np.float32), np.zeros((4, 4, d // 4), np.float32), R), rng


def test_blas_found():
    assert _lib.numpy_cblas() is not None


@pytest.mark.parametrize("d", [16, 128, 960])
def test_rows_bitwise_equal_per_query_rotate(d):
    q, rng = _quantizer(d)
    Y = (rng.normal(size=(300, d)) * 40).astype(np.float32)
    got = rotated_queries(q, Y)
    want = np.stack([np.asarray(q.rotate(Y[i:i + 1]), np.float32)[0] for i in range(Y.shape[0])])
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("ma", [1, 2, 3, 8, 64])
def test_blocks_bitwise_equal_per_query_rotate(ma):
    q, rng = _quantizer(128, seed=ma)
    res = (rng.normal(size=(50 * ma, 128)) * 40).astype(np.float32)
    got = _lib.rotate_rows(q, res, ma)
    assert got is not None
    want = np.concatenate([np.asarray(q.rotate(res[i * ma:(i + 1) * ma]), np.float32) for i in range(50)])
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_golden_opq_rotation():
    g = load_golden("opq_blobs")
    q = ArrayQuantizer(g["codebooks"], g["derived"], g["rotation"])
    got = rotated_queries(q, g["queries"])
    want = np.stack([(g["queries"][i:i + 1] @ g["rotation"]).astype(np.float32)[0]
                     for i in range(g["queries"].shape[0])])
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_custom_rotate_falls_back():
    class Custom(ArrayQuantizer):
        def rotate(self, X):
            return (X @ self.rotation_).astype(np.float32) + 0

    q, rng = _quantizer(16)
    c = Custom(q.codebooks_, q.derived_codebooks_, q.rotation_)
    assert _lib.rotate_rows(c, np.ones((4, 16), np.float32), 1) is None
