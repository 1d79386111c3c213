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


@pytest.mark.parametrize("world,env", [(3, {}), (2, {"DPQ_EXACT_LIMIT": "0", "DPQ_GUARD_SAMPLE": "16"}),
                                       (2, {"DPQ_SCAN_HIST": "1"}),
                                       (2, {"DPQ_SCAN_HIST": "1", "DPQ_EXACT_LIMIT": "0", "DPQ_EMIT_CAP": "64"})])
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


def _run_shards_dev(cb, der, codes, Y, r, r2, world):
    """Device-resident driver: per-shard streams, tensors exchanged in place."""
    import torch

    from paper_1905_06900_b200.shard import sharded_search_dev

    n = codes.shape[0]
    comm = ThreadComm(world)
    out = [None] * world
    errs = []
    engines = [GpuShardEngine(cb, der, codes[rk * n // world:(rk + 1) * n // world], rk * n // world, n, codes[:r2],
                              device=0) for rk in range(world)]

    def go(rank):
        try:
            comm.bind(rank)
            eng = engines[rank]
            with eng.context():
                y = eng.to_device(Y)
            d, i = sharded_search_dev(eng, comm, y, r, r2)
            with eng.context():
                out[rank] = (d.cpu().numpy(), i.cpu().numpy())
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
    torch.cuda.synchronize()
    return out


def _model(seed, m=4, k=1024, kbar=256, dsub=8, n=40000, nq=20):
    rng = np.random.default_rng(seed)
    cb = (rng.normal(size=(m, k, dsub)) * 3).astype(np.float32)
    der = np.stack([np.stack([cb[j][np.arange(k) % kbar == g].mean(axis=0) for g in range(kbar)])
                    for j in range(m)]).astype(np.float32)
    codes = rng.integers(0, k, size=(n, m)).astype(np.uint16)
    Y = (rng.normal(size=(nq, m * dsub)) * 3).astype(np.float32)
    return cb, der, codes, Y


@pytest.mark.parametrize("world,env", [(3, {}), (2, {"DPQ_EXACT_LIMIT": "0", "DPQ_GUARD_SAMPLE": "16"}),
                                       (2, {"DPQ_EXACT_LIMIT": "0", "DPQ_EMIT_CAP": "64"}),
                                       (3, {"DPQ_SCAN_HIST": "1"}),
                                       (2, {"DPQ_SCAN_HIST": "1", "DPQ_EXACT_LIMIT": "0", "DPQ_EMIT_CAP": "64"}),
                                       (2, {"DPQ_SCAN_HIST": "1", "DPQ_EXACT_LIMIT": "0", "DPQ_GUARD_SAMPLE": "16"})])
def test_sharded_device_protocol_equals_unsharded(world, env, monkeypatch):
    """dpq_shard_*_dev + in-place exchange + dpq_merge_topr_dev, including the
    flagged-redo path (tight guards from a 16-row sample; emit overflow)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cb, der, codes, Y = _model(12)
    r, r2 = 30, 500
    d0, i0 = O.flat_search(cb, der, codes, Y, r, "derived", r2)
    for d, i in _run_shards_dev(cb, der, codes, Y, r, r2, world):
        assert np.array_equal(i, i0)
        assert np.array_equal(d.view(np.uint64), d0.view(np.uint64))


@pytest.mark.parametrize("parts,r", [(2, 5), (3, 64), (8, 100), (5, 1)])
def test_merge_topr_dev_equals_host_merge(parts, r):
    import torch

    from paper_1905_06900_b200.shard import merge_topr

    rng = np.random.default_rng(parts * 100 + r)
    nq = 33
    pd = np.empty((parts, nq, r))
    pi = np.empty((parts, nq, r), np.int64)
    ids = rng.permutation(parts * nq * r * 4)[: parts * nq * r].reshape(parts, nq, r)
    for g in range(parts):
        for q in range(nq):
            d = rng.integers(0, 6, size=r).astype(np.float64) / 4  # heavy exact ties across parts
            npad = int(rng.integers(0, r + 1)) if q % 3 == 0 else 0
            d[r - npad:] = np.inf
            ii = ids[g, q].copy()
            ii[r - npad:] = -1
            o = np.lexsort((np.where(ii < 0, np.iinfo(np.int64).max, ii), d))
            pd[g, q], pi[g, q] = d[o], ii[o]
    want_d, want_i = merge_topr(list(pd), list(pi), r)
    cb, der, codes, _ = _model(1, n=100)
    eng = GpuShardEngine(cb, der, codes, 0, 100, codes[:10], device=0)
    with eng.context():
        md, mi = eng.merge_dev(torch.as_tensor(pd, device=eng.device), torch.as_tensor(pi, device=eng.device), r)
        md, mi = md.cpu().numpy(), mi.cpu().numpy()
    assert np.array_equal(mi, want_i)
    assert np.array_equal(md.view(np.uint64), want_d.view(np.uint64))


def test_sharded_flat_index_nccl_world1():
    """ShardedFlatIndex.search through real NCCL collectives (world size 1
    on this GPU): the public sharded API equals FlatIndex.search."""
    import socket

    import torch.distributed as dist

    from paper_1905_06900_b200.flat import ArrayQuantizer
    from paper_1905_06900_b200.shard import ShardedFlatIndex

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        cb, der, codes, Y = _model(13, nq=300)
        r, r2 = 20, 400
        q = ArrayQuantizer(cb, der)
        sidx = ShardedFlatIndex(q, codes, 0, codes.shape[0], codes[:r2], device=0, batch=128)
        d, i = sidx.search(Y, r, r2=r2)
        d1, i1 = FlatIndex.from_arrays(cb, der, codes).search(Y, r, mode="derived", r2=r2)
        assert np.array_equal(i, i1)
        assert np.array_equal(d.view(np.uint64), d1.view(np.uint64))
    finally:
        dist.destroy_process_group()


def _run_ivf_shards(g, Y, r, ma, r2, world, prefix_rows=4096, rotation=None):
    from paper_1905_06900_b200.flat import ArrayQuantizer
    from paper_1905_06900_b200.shard import ShardedIVFIndex

    comm = ThreadComm(world)
    out = [None] * world
    errs = []
    q = ArrayQuantizer(g["codebooks"], g["derived"], rotation)
    idxs = [ShardedIVFIndex(q, g["centers"], g["offsets"], g["sorted_codes"], g["sorted_ids"], rk, world, comm=comm,
                            prefix_rows=prefix_rows, device=0) for rk in range(world)]

    def go(rank):
        try:
            comm.bind(rank)
            out[rank] = idxs[rank].search(Y, r, ma=ma, r2=r2)
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


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["ivf_blobs", "ivf_opq"])
def test_ivf_list_split_shards_equal_reference(name, world):
    """IVF list-split sharding on the golden fixtures: every
    rank returns the reference's own IVFIndex.search result."""
    from conftest import load_golden

    g = load_golden(name)
    m = g["meta"]
    for d, i in _run_ivf_shards(g, g["queries"], m["r"], m["ma"], m["r2"], world, rotation=g.get("rotation")):
        assert np.array_equal(i, g["exp_derived_i"])
        assert np.array_equal(d.view(np.uint64), g["exp_derived_d"].view(np.uint64))


@pytest.mark.parametrize("env", [{}, {"DPQ_EXACT_LIMIT": "0", "DPQ_GUARD_SAMPLE": "8"}])
def test_ivf_list_split_random_equals_unsharded(env, monkeypatch):
    """Random IVF model with short and empty lists (some lists empty on some
    shards, so bound sources live on other shards) and a sampled-guard
    variant that forces the exact redo."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    from paper_1905_06900_b200.ivf import IVFIndex

    rng = np.random.default_rng(21)
    m, k, kbar, dsub, K, n = 4, 256, 16, 4, 24, 6000
    cb = (rng.normal(size=(m, k, dsub)) * 2).astype(np.float32)
    der = np.stack([np.stack([cb[j][np.arange(k) % kbar == g].mean(axis=0) for g in range(kbar)])
                    for j in range(m)]).astype(np.float32)
    centers = rng.normal(size=(K, m * dsub)).astype(np.float32) * 3
    sizes = rng.integers(0, 600, size=K)
    sizes[[2, 5, 11]] = [0, 1, 2]  # empty and tiny lists
    sizes = (sizes * n / max(1, sizes.sum())).astype(np.int64)
    offsets = np.zeros(K + 1, np.int64)
    offsets[1:] = np.cumsum(sizes)
    N = int(offsets[-1])
    g = {"codebooks": cb, "derived": der, "centers": centers, "offsets": offsets,
         "sorted_codes": rng.integers(0, k, size=(N, m)).astype(np.uint8),
         "sorted_ids": rng.permutation(N).astype(np.int64)}
    Y = (centers[rng.integers(K, size=40)] + rng.normal(size=(40, m * dsub))).astype(np.float32)
    r, ma, r2 = 15, 6, 300
    d0, i0 = IVFIndex.from_arrays(cb, der, centers, offsets, g["sorted_codes"], g["sorted_ids"]).search(
        Y, r, ma=ma, mode="derived", r2=r2)
    for world in (2, 4):
        for d, i in _run_ivf_shards(g, Y, r, ma, r2, world):
            assert np.array_equal(i, i0)
            assert np.array_equal(d.view(np.uint64), d0.view(np.uint64))
