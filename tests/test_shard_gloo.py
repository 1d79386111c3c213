"""Multi-rank host protocol of the sharded derived search (shard.py) on CPU:
world_size 2 over torch.distributed gloo, shard engines restated with the
oracle.  The merged result must equal the unsharded oracle bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import derived_search as O
from paper_1905_06900_b200.shard import TorchComm, merge_topr, sharded_search, sharded_search_dev
from shard_engines import OracleShardEngine


def _data(seed=0, n=3000, m=4, k=256, kbar=16, dsub=4, nq=9):
    rng = np.random.default_rng(seed)
    cb = (rng.normal(size=(m, k, dsub)) * 3).astype(np.float32)
    der = np.stack([np.stack([cb[j][np.arange(k) % kbar == g].mean(axis=0) for g in range(kbar)])
                    for j in range(m)]).astype(np.float32)
    codes = rng.integers(0, k, size=(n, m)).astype(np.uint8)
    Y = (rng.normal(size=(nq, m * dsub)) * 3).astype(np.float32)
    return cb, der, codes, Y


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, args, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cb, der, codes, Y, r, r2, sample, exact_limit, dev = args
    n = codes.shape[0]
    lo, hi = rank * n // world, (rank + 1) * n // world
    eng = OracleShardEngine(cb, der, codes[lo:hi], lo, n, codes[:max(r2, 1)], sample=sample,
                            exact_limit=exact_limit)
    if dev:  # the device-resident driver (tensors, in-place collectives, merge_dev)
        import torch

        d, i = sharded_search_dev(eng, TorchComm(), torch.as_tensor(Y), r, r2)
        d, i = d.numpy(), i.numpy()
    else:
        d, i = sharded_search(eng, TorchComm(), Y, r, r2)
    q.put((rank, d, i))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, args, q)) for rk in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return {rk: (d, i) for rk, d, i in out}


@pytest.mark.parametrize("dev", [False, True])
@pytest.mark.parametrize("sample,exact_limit", [(16384, 65536), (8, 0)])
def test_two_rank_gloo_equals_unsharded(sample, exact_limit, dev):
    cb, der, codes, Y = _data()
    r, r2 = 10, 200
    res = _run(2, (cb, der, codes, Y, r, r2, sample, exact_limit, dev))
    d0, i0 = O.flat_search(cb, der, codes, Y, r, "derived", r2)
    for rk in (0, 1):
        d, i = res[rk]
        assert np.array_equal(i, i0)
        assert np.array_equal(d.view(np.uint64), d0.view(np.uint64))


def test_merge_topr_ties_and_padding():
    d = [np.array([[1.0, 2.0, np.inf]]), np.array([[1.0, 1.5, np.inf]])]
    i = [np.array([[7, 3, -1]]), np.array([[5, 9, -1]])]
    md, mi = merge_topr(d, i, 4)
    assert mi.tolist() == [[5, 7, 9, 3]] and md.tolist() == [[1.0, 1.0, 1.5, 2.0]]
    md, mi = merge_topr([np.array([[np.inf, np.inf]])], [np.array([[-1, -1]])], 2)
    assert mi.tolist() == [[-1, -1]] and np.isinf(md).all()
