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

Two drivers of the same protocol:

* `sharded_search_dev` (the fast path): queries, histograms, flags and
  results stay in device memory; the phases only enqueue work on the shard's
  stream and the collectives run in place on that stream (NCCL), the merge
  is a device kernel (dpq_merge_topr_dev).  The only host synchronisation is
  reading the all-reduced flag byte at the end of the batch; a batch whose
  guard proved too tight or whose emit list overflowed on some shard is
  redone through the host driver.
* `sharded_search`: the host-buffer driver (numpy in and out between the
  phases), used for those rare redos and by the CPU protocol tests.

Both are engine- and transport-agnostic: `GpuShardEngine` drives libdpq;
`TorchComm` moves arrays/tensors with torch.distributed (NCCL on GPUs, gloo
for the CPU tests of this protocol).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .flat import rotated_queries


class GpuShardEngine:
    """One shard on one GPU: rows [row_base, row_base + len(codes)) of a
    database of n_global rows.  prefix_codes = the global first
    min(N, max r2) rows, replicated on every shard (qmax, twopass.py:83-84).
    All device work of the shard runs on `self.stream`."""

    def __init__(self, codebooks, derived, codes, row_base: int, n_global: int, prefix_codes, device: int = 0,
                 stream=None):
        import torch

        self.torch = torch
        self.handle = _lib.flat_create(codebooks, derived, codes, device=device, id_base=row_base,
                                       prefix_codes=prefix_codes)
        self.n_global = int(n_global)
        self.n_local = int(np.asarray(codes).shape[0])
        self.row_base = int(row_base)
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=self.device)
        self.handle.set_stream(self.stream.cuda_stream)
        self.sample_global = {}  # exact -> total sampled rows over the shards (all-reduced once)

    # ---- host-buffer protocol ------------------------------------------
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

    # ---- device protocol (enqueue only, on self.stream) -----------------
    def context(self):
        return self.torch.cuda.stream(self.stream)

    def to_device(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(a), device=self.device)

    def begin_dev(self, y, r2: int, exact: bool):
        torch = self.torch
        nq = y.shape[0]
        hist = torch.empty((nq, 256), dtype=torch.int32, device=self.device)
        ns = np.zeros(1, dtype=np.int64)
        _lib.check(_lib.lib().dpq_shard_begin_dev(self.handle.raw, _lib.ptr(y), nq, int(r2), self.n_global,
                                                  int(bool(exact)), _lib.ptr(hist), _lib.ptr(ns)), "shard_begin_dev")
        return hist, int(ns[0])

    def scan_dev(self, hist_sum, sample_global: int, r2: int, exact: bool):
        cand = self.torch.empty_like(hist_sum)
        _lib.check(_lib.lib().dpq_shard_scan_dev(self.handle.raw, _lib.ptr(hist_sum), self.n_global,
                                                 int(sample_global), int(r2), int(bool(exact)), _lib.ptr(cand)),
                   "shard_scan_dev")
        return cand

    def finish_dev(self, cand_sum, r: int, r2: int):
        torch = self.torch
        nq = cand_sum.shape[0]
        d = torch.empty((nq, r), dtype=torch.float64, device=self.device)
        i = torch.empty((nq, r), dtype=torch.int64, device=self.device)
        flags = torch.empty(nq, dtype=torch.uint8, device=self.device)
        _lib.check(_lib.lib().dpq_shard_finish_dev(self.handle.raw, _lib.ptr(cand_sum), int(r), int(r2),
                                                   _lib.ptr(d), _lib.ptr(i), _lib.ptr(flags)), "shard_finish_dev")
        return d, i, flags

    def merge_dev(self, parts_d, parts_i, r: int):
        torch = self.torch
        g, nq = parts_d.shape[0], parts_d.shape[1]
        d = torch.empty((nq, r), dtype=torch.float64, device=self.device)
        i = torch.empty((nq, r), dtype=torch.int64, device=self.device)
        _lib.check(_lib.lib().dpq_merge_topr_dev(self.handle.raw, _lib.ptr(parts_d), _lib.ptr(parts_i), g, nq,
                                                 int(r), _lib.ptr(d), _lib.ptr(i)), "merge_topr_dev")
        return d, i

    def search_dev(self, y, r: int, r2: int, comm=None):
        """Sharded derived search of device queries y (already rotated)."""
        return sharded_search_dev(self, comm or self.comm, y, r, r2)


class TorchComm:
    """All-reduce / all-gather over a torch.distributed process group.
    Host arrays (the host protocol) travel through tensors on `device` (cuda
    for NCCL, cpu for gloo); tensors (the device protocol) are reduced in
    place on the current stream."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        if device is None:
            device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        self.device = device
        self.world = dist.get_world_size(group)

    # ---- host arrays ----------------------------------------------------
    def _t(self, a):
        return self.torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def allreduce_sum(self, a: np.ndarray) -> np.ndarray:
        t = self._t(np.asarray(a).astype(np.int64))
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

    # ---- tensors, in place ----------------------------------------------
    def sum_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def max_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t

    def gather_stack(self, t):
        """(world, *t.shape) tensor of every rank's t."""
        out = self.torch.empty((self.world, *t.shape), dtype=t.dtype, device=t.device)
        self.dist.all_gather(list(out.unbind(0)), t.contiguous(), group=self.group)
        return out


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
    """Derived search of yr (already rotated) over all shards, host-buffer
    driver.  Returns the same (dists, ids) on every rank."""
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


def sharded_search_dev(engine, comm, y, r: int, r2: int):
    """Device-resident driver of the same protocol: y is a (nq, d) tensor on
    the engine's device (already rotated); returns (dists, ids) tensors,
    identical on every rank.  Collectives run in place on the engine's
    stream; the host waits only for the all-reduced flags at the end."""
    if r > r2:
        raise ValueError(f"r={r} must not exceed r2={r2}")
    with engine.context():
        hist, ns = engine.begin_dev(y, r2, False)
        if False not in engine.sample_global:  # total sampled rows: fixed per shard layout, reduced once
            engine.sample_global[False] = int(comm.allreduce_sum(np.array([ns], dtype=np.int64))[0])
        comm.sum_(hist)
        cand = engine.scan_dev(hist, engine.sample_global[False], r2, False)
        comm.sum_(cand)
        d, i, flags = engine.finish_dev(cand, r, r2)
        parts_d = comm.gather_stack(d)
        parts_i = comm.gather_stack(i)
        fl = comm.max_(flags.to(engine.torch.int32).max().reshape(1))
        md, mi = engine.merge_dev(parts_d, parts_i, r)
        redo = int(fl.item()) != 0  # the batch's only host synchronisation
    if redo:  # a guard proved too tight or an emit list overflowed on some shard: redo through the host driver
        yh = y.detach().cpu().numpy()
        dh, ih = sharded_search(engine, comm, yh, r, r2)
        md, mi = engine.to_device(dh), engine.to_device(ih)
    return md, mi


class ShardedFlatIndex:
    """FlatIndex.search(mode="derived") over a database split across ranks.

    Each rank constructs it with its own row shard; `search` is collective
    (every rank calls it with the same queries) and returns the global
    result on every rank."""

    def __init__(self, quantizer, codes_shard, row_base: int, n_global: int, prefix_codes, comm=None,
                 device: int = 0, batch: int = 1024):
        self.quantizer = quantizer
        self.comm = comm if comm is not None else TorchComm()
        self.batch = int(batch)
        self.engine = GpuShardEngine(quantizer.codebooks_, quantizer.derived_codebooks_, codes_shard, row_base,
                                     n_global, prefix_codes, device=device)
        self.engine.comm = self.comm

    def search(self, Y, r: int, mode: str = "derived", r2=None):
        if mode != "derived":
            raise ValueError("ShardedFlatIndex supports mode='derived'")
        if r2 is None:
            raise ValueError("derived mode requires r2")
        Y = _lib.query_array(Y)
        yr = rotated_queries(self.quantizer, Y)
        if yr.shape[0] == 0:
            return np.full((0, r), np.inf), np.full((0, r), -1, dtype=np.int64)
        eng = self.engine
        out_d = np.empty((yr.shape[0], r), np.float64)
        out_i = np.empty((yr.shape[0], r), np.int64)
        with eng.context():
            ydev = eng.to_device(yr)
        for s in range(0, yr.shape[0], self.batch):
            d, i = sharded_search_dev(eng, self.comm, ydev[s:s + self.batch], r, r2)
            with eng.context():
                out_d[s:s + self.batch] = d.cpu().numpy()
                out_i[s:s + self.batch] = i.cpu().numpy()
        return out_d, out_i



# --------------------------------------------------------------- IVF --------

def split_lists(offsets, sorted_codes, sorted_ids, rank: int, world: int):
    """This shard's slice of every inverted list (each list cut
    evenly across the shards, cell order kept): local offsets (K+1), codes,
    GLOBAL ids."""
    offsets = np.asarray(offsets, dtype=np.int64)
    lens = np.diff(offsets)
    lo = offsets[:-1] + lens * rank // world
    hi = offsets[:-1] + lens * (rank + 1) // world
    loc = np.zeros_like(offsets)
    loc[1:] = np.cumsum(hi - lo)
    rows = np.concatenate([np.arange(a, b, dtype=np.int64) for a, b in zip(lo, hi)]) if len(lo) else \
        np.empty(0, np.int64)
    return loc, np.ascontiguousarray(np.asarray(sorted_codes)[rows]), np.ascontiguousarray(
        np.asarray(sorted_ids)[rows])


def list_prefixes(offsets, sorted_codes, rows: int):
    """First min(rows, len) rows of every global list, concatenated, with
    their row offsets (the replicated qmax prefixes, ivf.py:205-217)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    take = np.minimum(np.diff(offsets), rows)
    pre_off = np.zeros_like(offsets)
    pre_off[1:] = np.cumsum(take)
    idx = np.concatenate([np.arange(o, o + t, dtype=np.int64) for o, t in zip(offsets[:-1], take)]) if len(take) \
        else np.empty(0, np.int64)
    return np.ascontiguousarray(np.asarray(sorted_codes)[idx]), pre_off


class GpuIvfShardEngine:
    """One list-split IVF shard on one GPU (dpq_ivf_set_shard)."""

    def __init__(self, codebooks, derived, centers, offsets, sorted_codes, sorted_ids, rank: int, world: int,
                 prefix_rows: int = 4096, device: int = 0):
        loc, codes, ids = split_lists(offsets, sorted_codes, sorted_ids, rank, world)
        self.handle = _lib.ivf_create(codebooks, derived, centers, loc, codes, ids, device=device)
        cb = _lib.code_bytes_of(np.asarray(sorted_codes))
        pre, pre_off = list_prefixes(offsets, sorted_codes, prefix_rows)
        pre = np.ascontiguousarray(pre, dtype=np.uint8 if cb == 1 else np.uint16)
        g_off = np.ascontiguousarray(offsets, dtype=np.int64)
        _lib.check(_lib.lib().dpq_ivf_set_shard(self.handle.raw, _lib.ptr(g_off), _lib.ptr(pre), _lib.ptr(pre_off),
                                                int(prefix_rows)), "ivf_set_shard")
        self.n_local = int(ids.shape[0])

    def probe(self, Y: np.ndarray, ma: int) -> np.ndarray:
        cells = np.empty((Y.shape[0], ma), np.int64)
        _lib.check(_lib.lib().dpq_ivf_probe(self.handle.raw, _lib.ptr(Y), Y.shape[0], int(ma), _lib.ptr(cells)),
                   "ivf_probe")
        return cells

    def begin(self, Y, ma, r2, exact, res_rot=None, cells=None):
        nq = Y.shape[0]
        hist = np.zeros((nq, 256), np.int32)
        ns = np.zeros(nq, np.int64)
        nr = np.zeros(nq, np.int64)
        _lib.check(_lib.lib().dpq_ivf_shard_begin(self.handle.raw, _lib.ptr(Y), nq, int(ma), int(r2), int(bool(exact)),
                                                  _lib.ptr(res_rot), _lib.ptr(cells), _lib.ptr(hist), _lib.ptr(ns),
                                                  _lib.ptr(nr)), "ivf_shard_begin")
        return hist, ns, nr

    def scan(self, hist_sum, ns_sum, nr, r2):
        hist_sum = np.ascontiguousarray(hist_sum, dtype=np.int32)
        ns_sum = np.ascontiguousarray(ns_sum, dtype=np.int64)
        nr = np.ascontiguousarray(nr, dtype=np.int64)
        cand = np.zeros_like(hist_sum)
        _lib.check(_lib.lib().dpq_ivf_shard_scan(self.handle.raw, _lib.ptr(hist_sum), _lib.ptr(ns_sum), _lib.ptr(nr),
                                                 int(r2), _lib.ptr(cand)), "ivf_shard_scan")
        return cand

    def finish(self, cand_sum, r, r2):
        cand_sum = np.ascontiguousarray(cand_sum, dtype=np.int32)
        nq = cand_sum.shape[0]
        d = np.empty((nq, r), np.float64)
        i = np.empty((nq, r), np.int64)
        need = np.zeros(nq, np.uint8)
        _lib.check(_lib.lib().dpq_ivf_shard_finish(self.handle.raw, _lib.ptr(cand_sum), int(r), int(r2), _lib.ptr(d),
                                                   _lib.ptr(i), _lib.ptr(need)), "ivf_shard_finish")
        return d, i, need.astype(bool)


def sharded_ivf_search(engine, comm, Y: np.ndarray, r: int, ma: int, r2: int, res_rot=None, cells=None):
    """IVFIndex.search(mode="derived") over list-split shards (ivf.py:195-277):
    one candidate pool per query across the probed lists of every shard,
    refine in each candidate's own cell frame, merge by (dist, id)."""
    if r > r2:
        raise ValueError(f"r={r} must not exceed r2={r2}")
    Y = np.ascontiguousarray(Y, dtype=np.float32)
    exact = False
    for _ in range(2):
        hist, ns, nr = engine.begin(Y, ma, r2, exact, res_rot, cells)
        hist_sum = comm.allreduce_sum(hist)
        ns_sum = comm.allreduce_sum(ns)
        cand = engine.scan(hist_sum, ns_sum, nr, r2)
        cand_sum = comm.allreduce_sum(cand)
        d, i, need = engine.finish(cand_sum, r, r2)
        if not comm.allreduce_max(int(need.any())):
            break
        exact = True  # a guard proved too tight on some query: redo with exact histograms
    return merge_topr(comm.allgather(d), comm.allgather(i), r)


class ShardedIVFIndex:
    """IVFIndex.search(mode="derived") over an IVF index whose every list is
    split across ranks.  Each rank constructs it from the same global arrays
    (it keeps only its slices); `search` is collective and returns the global
    result on every rank."""

    def __init__(self, quantizer, centers, offsets, sorted_codes, sorted_ids, rank: int, world: int, comm=None,
                 prefix_rows: int = 4096, device: int = 0, batch: int = 4096):
        self.quantizer = quantizer
        self.centers_ = np.ascontiguousarray(centers, dtype=np.float32)
        self.comm = comm if comm is not None else TorchComm()
        self.batch = int(batch)
        self.engine = GpuIvfShardEngine(quantizer.codebooks_, quantizer.derived_codebooks_, self.centers_, offsets,
                                        sorted_codes, sorted_ids, rank, world, prefix_rows=prefix_rows, device=device)

    def search(self, Y, r: int, ma: int = 8, mode: str = "derived", r2=None):
        if mode != "derived":
            raise ValueError("ShardedIVFIndex supports mode='derived'")
        if r2 is None:
            raise ValueError("derived mode requires r2")
        Y = _lib.query_array(Y)
        if not (1 <= ma <= self.centers_.shape[0]):
            raise ValueError(f"ma must be in [1, {self.centers_.shape[0]}], got {ma}")
        out_d, out_i = [], []
        for s in range(0, Y.shape[0], self.batch):
            Yb = np.ascontiguousarray(Y[s:s + self.batch])
            res_rot = cells = None
            if getattr(self.quantizer, "rotation_", None) is not None:  # OPQ: (ma, d) rotate per query (ivf.py:202)
                cells = self.engine.probe(Yb, ma)
                res = (Yb[:, None, :] - self.centers_[cells]).reshape(-1, Yb.shape[1])
                rot = _lib.rotate_rows(self.quantizer, res, ma)
                if rot is None:
                    rot = np.concatenate([np.asarray(self.quantizer.rotate(res[q * ma:(q + 1) * ma]), np.float32)
                                          for q in range(Yb.shape[0])])
                res_rot = np.ascontiguousarray(rot, dtype=np.float32)
            d, i = sharded_ivf_search(self.engine, self.comm, Yb, r, ma, r2, res_rot, cells)
            out_d.append(d)
            out_i.append(i)
        if not out_d:
            return np.full((0, r), np.inf), np.full((0, r), -1, dtype=np.int64)
        return np.concatenate(out_d), np.concatenate(out_i)
