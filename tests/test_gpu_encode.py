"""Tensor-core encoder (dpq_encode, tcgen05 3xTF32 GEMM + row argmin) vs the
reference encoder (quantizer.py:75-83 -> clustering.py:53-77).

* Pinned: the config-1-shape golden codes were produced by the reference's
  own encoder (tests/golden/make_golden.py); its codebooks are integer SIFT
  points, so every distance is an exact integer in both implementations and
  the codes must match bit for bit.
* Float data (3xTF32 path): agreement with the exact float64 argmin, where a
  disagreement is allowed only at a near-tie (the reference's cross term is
  an f32 BLAS GEMM, itself rounding-dependent).
* Edge shapes: k not a multiple of the 128-centroid tile, dsub < 32, row
  counts around the 256-row unit, exact duplicate centroids (lowest index).
"""

import numpy as np
import pytest

from paper_1905_06900_b200 import _lib, datagen

pytestmark = pytest.mark.gpu


def exact_argmin(x, cb):
    """f64 argmin per subspace, ties to the lowest index; also the gap
    d(chosen) - d(best) helper."""
    m, k, dsub = cb.shape
    out = np.empty((x.shape[0], m), np.int64)
    d2s = []
    for j in range(m):
        xs = x[:, j * dsub:(j + 1) * dsub].astype(np.float64)
        c = cb[j].astype(np.float64)
        d2 = (xs * xs).sum(1)[:, None] - 2.0 * xs @ c.T + (c * c).sum(1)[None, :]
        out[:, j] = np.argmin(d2, axis=1)
        d2s.append(d2)
    return out, d2s


def test_config1_codes_bitwise_vs_reference_encoder(c1_golden):
    st = datagen.seed_streams(datagen.SEED)
    centres = datagen.sift_centres(st["centres"])
    X = datagen.sift_like(st["database"], centres, 100_000)
    enc = _lib.Encoder(c1_golden["codebooks"], device=0)
    codes = enc.encode(X)
    assert codes.dtype == np.uint16 and codes.shape == (100_000, 4)
    assert np.array_equal(codes, c1_golden["codes"])


@pytest.mark.parametrize("m,k,dsub,n,scale", [(2, 4096, 32, 3000, 1.0), (3, 1000, 24, 777, 50.0),
                                              (1, 8192, 32, 1500, 0.01),
                                              # K-chunked path (dsub > 32): configs[4]'s dsub = 120 and the
                                              # IVF coarse assignment (m = 1, d = 128, K = 8192)
                                              (2, 4096, 120, 2000, 1.0), (1, 8192, 128, 1500, 30.0),
                                              (3, 700, 48, 999, 0.5)])
def test_float_data_matches_exact_argmin_up_to_near_ties(m, k, dsub, n, scale):
    rng = np.random.default_rng(k + n)
    cb = (rng.normal(size=(m, k, dsub)) * scale).astype(np.float32)
    x = (rng.normal(size=(n, m * dsub)) * scale).astype(np.float32)
    got = _lib.Encoder(cb).encode(x).astype(np.int64)
    want, d2s = exact_argmin(x, cb)
    agree = got == want
    assert agree.mean() >= 0.995, agree.mean()
    for j in range(m):
        bad = np.flatnonzero(~agree[:, j])
        if bad.size:
            d2 = d2s[j]
            gap = d2[bad, got[bad, j]] - d2[bad, want[bad, j]]
            ref = (x[bad, j * dsub:(j + 1) * dsub].astype(np.float64) ** 2).sum(1) + d2[bad, want[bad, j]]
            assert np.all(gap <= 1e-5 * np.maximum(ref, 1e-30) + 1e-6 * scale * scale), (gap, ref)


@pytest.mark.parametrize("k,dsub,n", [(16, 8, 1), (200, 30, 257), (256, 5, 1000), (65536, 32, 300)])
def test_integer_data_exact(k, dsub, n):
    rng = np.random.default_rng(k * 7 + dsub)
    m = 2
    cb = rng.integers(0, 256, size=(m, k, dsub)).astype(np.float32)
    x = rng.integers(0, 256, size=(n, m * dsub)).astype(np.float32)
    got = _lib.Encoder(cb).encode(x).astype(np.int64)
    want, _ = exact_argmin(x, cb)
    assert np.array_equal(got, want)


def test_duplicate_centroids_lowest_index():
    rng = np.random.default_rng(5)
    k, dsub = 512, 32
    cb = rng.integers(0, 64, size=(1, k, dsub)).astype(np.float32)
    cb[0, 300] = cb[0, 7]
    cb[0, 450] = cb[0, 7]
    cb[0, 129] = cb[0, 128]
    x = np.stack([cb[0, 300], cb[0, 129], cb[0, 450] + 0.0]).astype(np.float32)
    got = _lib.Encoder(cb).encode(x)[:, 0]
    assert got.tolist() == [7, 128, 7]


def test_device_entry_and_errors():
    import torch

    rng = np.random.default_rng(9)
    cb = rng.integers(0, 256, size=(4, 1024, 32)).astype(np.float32)
    x = rng.integers(0, 256, size=(5000, 160)).astype(np.float32)  # row stride 160 > m*dsub
    enc = _lib.Encoder(cb)
    xt = torch.as_tensor(x, device="cuda")
    codes = torch.empty((5000, 4), dtype=torch.int32, device="cuda")
    enc.encode_dev(xt, codes)
    torch.cuda.synchronize()
    want, _ = exact_argmin(np.ascontiguousarray(x[:, :128]), cb)
    assert np.array_equal(codes.cpu().numpy(), want)
    with pytest.raises(ValueError):
        _lib.Encoder(np.zeros((1, 16, 140), np.float32))
    with pytest.raises(ValueError):
        enc.encode(np.zeros((3, 100), np.float32))


def test_duplicate_centroids_lowest_index_chunked():
    rng = np.random.default_rng(6)
    k, dsub = 1024, 100
    cb = rng.normal(size=(1, k, dsub)).astype(np.float32)
    cb[0, 900] = cb[0, 3]
    cb[0, 513] = cb[0, 512]
    x = np.stack([cb[0, 900], cb[0, 513], cb[0, 3]]).astype(np.float32)
    got = _lib.Encoder(cb).encode(x)[:, 0]
    assert got.tolist() == [3, 512, 3]


def test_gist_like_codes_chunked():
    """configs[4] shape (8 x 65536 x 120) on GIST-like data: the tensor-core
    codes agree with the exact f64 argmin except at f32 near-ties."""
    rng = np.random.default_rng(8)
    centres = rng.uniform(0, 1, size=(64, 120))
    cb = np.clip(centres[rng.integers(64, size=(8, 65536))] + rng.normal(0, 0.05, size=(8, 65536, 120)), 0, 1)
    cb = cb.astype(np.float32)
    x = np.clip(centres[rng.integers(64, size=(400, 8))].reshape(400, 960) + rng.normal(0, 0.05, size=(400, 960)),
                0, 1).astype(np.float32)
    got = _lib.Encoder(cb).encode(x).astype(np.int64)
    want, d2s = exact_argmin(x, cb)
    agree = got == want
    assert agree.mean() >= 0.99, agree.mean()
    for j in range(8):
        bad = np.flatnonzero(~agree[:, j])
        if bad.size:
            gap = d2s[j][bad, got[bad, j]] - d2s[j][bad, want[bad, j]]
            assert np.all(gap <= 1e-4), gap
