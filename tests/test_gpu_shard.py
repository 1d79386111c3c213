"""The GPU split API (dpq_shard_*) driven by the real multi-rank protocol
(shard.sharded_search): 3 shards as threads on one GPU exchanging through an
in-process comm (kernels never wait on each other).  Bar: bit-exact vs the
unsharded oracle and vs the unsharded GPU search."""

import threading

import numpy as np
import pytest

from oracle import derived_search as O
from paper_1905_06900_b200.flat import FlatIndex
from paper_1905_06900_b200.shard import GpuShardEngine, sharded_search
from shard_engines import ThreadComm

pytestmark = pytest.mark.gpu


def _run_shards(cb, der, codes, Y, r, r2, world):
    n = codes.shape[0]
    comm = ThreadComm(world)
    out = [None] * world
    errs = []

    def go(rank):
        try:
            comm.bind(rank)
            lo, hi = rank * n // world, (rank + 1) * n // world
            eng = GpuShardEngine(cb, der, codes[lo:hi], lo, n, codes[:r2], device=0)
            out[rank] = sharded_search(eng, comm, Y, r, r2)
        except Exception as exc:  # pragma: no cover
            errs.append(exc)
            comm.bar.abort()

    ts = [threading.Thread(target=go, args=(rk,)) for rk in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("world,env", [(3, {}), (2, {"DPQ_EXACT_LIMIT": "0", "DPQ_GUARD_SAMPLE": "16"})])
def test_sharded_gpu_equals_unsharded(world, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(11)
    m, k, kbar, dsub, n = 4, 1024, 256, 8, 40000
    cb = (rng.normal(size=(m, k, dsub)) * 3).astype(np.float32)
    der = np.stack([np.stack([cb[j][np.arange(k) % kbar == g].mean(axis=0) for g in range(kbar)])
                    for j in range(m)]).astype(np.float32)
    codes = rng.integers(0, k, size=(n, m)).astype(np.uint16)
    Y = (rng.normal(size=(20, m * dsub)) * 3).astype(np.float32)
    r, r2 = 30, 500
    d0, i0 = O.flat_search(cb, der, codes, Y, r, "derived", r2)
    d1, i1 = FlatIndex.from_arrays(cb, der, codes).search(Y, r, mode="derived", r2=r2)
    assert np.array_equal(i0, i1)
    for d, i in _run_shards(cb, der, codes, Y, r, r2, world):
        assert np.array_equal(i, i0)
        assert np.array_equal(d.view(np.uint64), d0.view(np.uint64))
