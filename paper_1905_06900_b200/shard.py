"""Database-sharded derived search across GPUs (north_star (v)).

The flat database is split into contiguous row shards, one per rank/GPU.
Per query batch the ranks run the three-phase split API of libdpq
(include/dpq.h, dpq_shard_*) with two histogram all-reduces between the
phases and a final all-gather of the per-shard top-r:

  begin  -> per-shard sample histograms   --all-reduce(sum)-->  guards
  scan   -> per-shard candidate histograms --all-reduce(sum)-->  global b*
  finish -> per-shard exact top-r with global ids --all-gather--> merge

Every rank computes the same guard and the same b* from identical summed
histograms, so the union of the shards' candidates is exactly the unsharded
candidate set {score <= b*} (twopass.py:171-201, 295-302) and the merged
top-r by (dist, id) equals the unsharded result bit for bit.

The orchestration (`sharded_search`) is engine- and transport-agnostic:
`GpuShardEngine` drives libdpq; `TorchComm` moves the small arrays with
torch.distributed (NCCL on GPUs, gloo for the CPU tests of this protocol).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .flat import rotated_queries


class GpuShardEngine:
    """One shard on one GPU: rows [row_base, row_base + len(codes)) of a
    database of n_global rows.  prefix_codes = the global first
    min(N, max r2) rows, replicated on every shard (qmax, twopass.py:83-84)."""

    def __init__(self, codebooks, derived, codes, row_base: int, n_global: int, prefix_codes, device: int = 0):
        self.handle = _lib.flat_create(codebooks, derived, codes, device=device, id_base=row_base,
                                       prefix_codes=prefix_codes)
        self.n_global = int(n_global)
        self.n_local = int(np.asarray(codes).shape[0])
        self.row_base = int(row_base)

    def begin(self, yr: np.ndarray, r2: int, exact: bool):
        nq = yr.shape[0]
        hist = np.zeros((nq, 256), dtype=np.int32)
        ns = np.zeros(1, dtype=np.int64)
        _lib.check(_lib.lib().dpq_shard_begin(self.handle.raw, _lib.ptr(yr), nq, int(r2), self.n_global,
                                              int(bool(exact)), _lib.ptr(hist), _lib.ptr(ns)), "shard_begin")
        return hist, int(ns[0])

    def scan(self, hist_sum: np.ndarray, sample_global: int, r2: int, exact: bool):
        hist_sum = np.ascontiguousarray(hist_sum, dtype=np.int32)
        cand = np.zeros_like(hist_sum)
        _lib.check(_lib.lib().dpq_shard_scan(self.handle.raw, _lib.ptr(hist_sum), self.n_global, int(sample_global),
                                             int(r2), int(bool(exact)), _lib.ptr(cand)), "shard_scan")
        return cand

    def finish(self, cand_sum: np.ndarray, r: int, r2: int):
        cand_sum = np.ascontiguousarray(cand_sum, dtype=np.int32)
        nq = cand_sum.shape[0]
        d = np.empty((nq, r), dtype=np.float64)
        i = np.empty((nq, r), dtype=np.int64)
        need = np.zeros(nq, dtype=np.uint8)
        _lib.check(_lib.lib().dpq_shard_finish(self.handle.raw, _lib.ptr(cand_sum), int(r), int(r2), _lib.ptr(d),
                                               _lib.ptr(i), _lib.ptr(need)), "shard_finish")
        return d, i, need.astype(bool)


class TorchComm:
    """Sum / max all-reduce and all-gather of small numpy arrays over a
    torch.distributed process group (device = cuda for NCCL, cpu for gloo)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        if device is None:
            device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        self.device = device
        self.world = dist.get_world_size(group)

    def _t(self, a):
        return self.torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def allreduce_sum(self, a: np.ndarray) -> np.ndarray:
        t = self._t(a.astype(np.int64))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()

    def allreduce_max(self, x: int) -> int:
        t = self._t(np.array([x], dtype=np.int64))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(t.cpu().numpy()[0])

    def allgather(self, a: np.ndarray) -> list:
        t = self._t(a)
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy() for o in out]


def merge_topr(dist_parts, id_parts, r: int):
    """Exact top-r by (dist, id) of per-shard top-r lists (search.py:73-88);
    rows padded with (+inf, -1) like pack_results (flat.py:16-29)."""
    d = np.concatenate(dist_parts, axis=1)
    i = np.concatenate(id_parts, axis=1)
    pad = i < 0
    i_key = np.where(pad, np.iinfo(np.int64).max, i)
    o1 = np.argsort(i_key, axis=1, kind="stable")
    d1 = np.take_along_axis(d, o1, 1)
    o2 = np.argsort(d1, axis=1, kind="stable")
    order = np.take_along_axis(o1, o2, 1)[:, :r]
    return np.take_along_axis(d, order, 1), np.take_along_axis(i, order, 1)


def sharded_search(engine, comm, yr: np.ndarray, r: int, r2: int):
    """Derived search of yr (already rotated) over all shards.  Returns the
    same (dists, ids) on every rank."""
    if r > r2:
        raise ValueError(f"r={r} must not exceed r2={r2}")
    yr = np.ascontiguousarray(yr, dtype=np.float32)
    exact = False
    for _ in range(2):
        hist, ns = engine.begin(yr, r2, exact)
        hist_sum = comm.allreduce_sum(hist)
        ns_sum = int(comm.allreduce_sum(np.array([ns], dtype=np.int64))[0])
        cand = engine.scan(hist_sum, ns_sum, r2, exact)
        cand_sum = comm.allreduce_sum(cand)
        d, i, need = engine.finish(cand_sum, r, r2)
        if not comm.allreduce_max(int(need.any())):
            break
        exact = True  # a guard proved too tight on some query: redo exactly
    return merge_topr(comm.allgather(d), comm.allgather(i), r)


class ShardedFlatIndex:
    """FlatIndex.search(mode="derived") over a database split across ranks.

    Each rank constructs it with its own row shard; `search` is collective
    (every rank calls it with the same queries) and returns the global
    result on every rank."""

    def __init__(self, quantizer, codes_shard, row_base: int, n_global: int, prefix_codes, comm,
                 device: int = 0):
        self.quantizer = quantizer
        self.comm = comm
        self.engine = GpuShardEngine(quantizer.codebooks_, quantizer.derived_codebooks_, codes_shard, row_base,
                                     n_global, prefix_codes, device=device)

    def search(self, Y, r: int, mode: str = "derived", r2=None, batch: int = 1024):
        if mode != "derived":
            raise ValueError("ShardedFlatIndex supports mode='derived'")
        if r2 is None:
            raise ValueError("derived mode requires r2")
        Y = np.ascontiguousarray(Y, dtype=np.float32)
        yr = rotated_queries(self.quantizer, Y)
        out_d, out_i = [], []
        for s in range(0, yr.shape[0], batch):
            d, i = sharded_search(self.engine, self.comm, yr[s:s + batch], r, r2)
            out_d.append(d)
            out_i.append(i)
        if not out_d:
            return np.full((0, r), np.inf), np.full((0, r), -1, dtype=np.int64)
        return np.concatenate(out_d), np.concatenate(out_i)
