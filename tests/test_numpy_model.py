"""Re-check, on whatever host runs the suite, the two numpy behaviours the
GPU kernels reproduce bit-for-bit ("re-check on the GPU
box host"): the float32 pairwise row sum and the NEP 50 float32 comparison.
"""

import numpy as np

F = np.float32


def pairwise_model(s):
    """numpy pairwise_sum model implemented by dpq_device.cuh:pw_sqdist."""
    n = len(s)
    if n < 8:
        res = F(-0.0)
        for x in s:
            res = F(res + x)
        return res
    if n <= 128:
        r = [s[i] for i in range(8)]
        lim = n - n % 8
        for i in range(8, lim, 8):
            for j in range(8):
                r[j] = F(r[j] + s[i + j])
        res = F(F(F(r[0] + r[1]) + F(r[2] + r[3])) + F(F(r[4] + r[5]) + F(r[6] + r[7])))
        for i in range(lim, n):
            res = F(res + s[i])
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return F(pairwise_model(s[:n2]) + pairwise_model(s[n2:]))


def test_row_sum_is_pairwise_8():
    rng = np.random.default_rng(0)
    for d in list(range(1, 140)) + [200, 256, 480, 960]:
        rows = (rng.normal(size=(12, d)) * rng.uniform(0.1, 100)).astype(np.float32)
        v = rng.normal(size=d).astype(np.float32)
        diff = rows - v
        sq = diff * diff
        ref = sq.sum(axis=1)
        mine = np.array([pairwise_model(list(sq[i])) for i in range(rows.shape[0])], dtype=np.float32)
        assert np.array_equal(ref.view(np.uint32), mine.view(np.uint32)), d


def test_nep50_float32_comparison():
    # a value above qmax in f64 but equal to float32(qmax) is NOT saturated
    qmax = 1.0 + 2.0 ** -30          # rounds to 1.0 in float32
    tables = np.array([1.0], dtype=np.float32)
    assert not bool((tables > qmax)[0])
    assert float(np.float32(qmax)) == 1.0
