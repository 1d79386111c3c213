"""GPU exact ground truth: the rank-0 nearest neighbour
the bench's Recall@100 uses (workloads.StreamingTruth: fp32 GEMM shortlist
over streamed chunks + f64 re-rank, ties to the lower id; train.exact_nn_gpu)
equals the reference's brute force exact_nn (evaluation.py:28-62) on
subsamples of the bench generators."""

import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import derived_search as O
from paper_1905_06900_b200 import datagen, workloads

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


def _ref_exact_nn():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    try:
        from derivedpq.evaluation import exact_nn
        return exact_nn
    except ImportError:
        return None


@pytest.mark.parametrize("kind,n,nq", [("sift", 150_000, 300), ("gist", 20_000, 64)])
def test_streaming_truth_equals_exact_nn(kind, n, nq):
    import torch

    st = datagen.seed_streams(7)
    if kind == "sift":
        c = datagen.sift_centres(st["centres"])
        X = datagen.sift_like(st["database"], c, n)
        Y = datagen.sift_like(st["queries"], c, nq)
    else:
        c = datagen.gist_centres(st["centres"])
        X = datagen.gist_like(st["database"], c, n)
        Y = datagen.gist_like(st["queries"], c, nq)
    X[17] = X[3]  # exact duplicate rows: the tie goes to the lower id
    Y[0] = X[3]
    dev = torch.device("cuda", 0)
    tr = workloads.StreamingTruth(Y, dev)
    xt = torch.as_tensor(X, device=dev)
    for s in range(0, n, 40_000):  # streamed in chunks like the bench's database
        tr.update(s, xt[s:s + 40_000])
    _, got = tr.result()
    want = O.exact_nn(X, Y, 1)[:, 0]
    assert np.array_equal(got, want)
    assert got[0] == 3
    ref = _ref_exact_nn()
    if ref is not None:
        assert np.array_equal(got, ref(X, Y, 1)[:, 0].astype(np.int64))
    from paper_1905_06900_b200 import train

    assert np.array_equal(train.exact_nn_gpu(xt, torch.as_tensor(Y, device=dev), depth=1)[:, 0], want)
