"""Test-only shard engine: the dpq_shard_* contract (include/dpq.h)
restated with the CPU oracle, so the multi-rank host protocol in
paper_1905_06900_b200/shard.py can be checked on CPU (gloo) exactly as the
GPU engine is driven on B200s."""

import contextlib
import math
import threading

import numpy as np
import torch

from oracle import derived_search as O


def guard_from_hist(hist, r2, lam, exact):
    """k_guard (dpq_kernels.cuh)."""
    target = float(r2) if exact else lam + 3.0 * math.sqrt(lam) + 4.0
    cum = np.cumsum(hist[:, :255], axis=1)
    out = np.full(hist.shape[0], 254, dtype=np.int64)
    for q in range(hist.shape[0]):
        hit = np.flatnonzero(cum[q] >= target)
        if hit.size:
            out[q] = hit[0]
    return out


class OracleShardEngine:
    def __init__(self, codebooks, derived, codes, row_base, n_global, prefix_codes, sample=16384,
                 exact_limit=65536):
        self.cb, self.der, self.codes = codebooks, derived, np.asarray(codes)
        self.base, self.n_global, self.prefix = row_base, n_global, np.asarray(prefix_codes)
        self.sample, self.exact_limit = sample, exact_limit
        self.sample_global = {}

    def begin(self, yr, r2, exact):
        self.yr = yr
        self.scores = []
        n = self.codes.shape[0]
        ex = exact or self.n_global <= self.exact_limit
        ns = 0 if n == 0 else (n if ex else min(n, self.sample))
        stride = n // ns if ns else 1
        hist = np.zeros((yr.shape[0], 256), dtype=np.int64)
        for q, y in enumerate(yr):
            small = O.lookup_tables(y, self.der)
            qt = O.quantize_small(small, self.prefix[: min(r2, self.n_global)], r2)
            s = O.low_scores(self.codes, qt) if n else np.empty(0, np.uint8)
            self.scores.append(s)
            samp = s[np.arange(ns) * stride]
            hist[q] = np.bincount(samp[samp < 255], minlength=256)
        return hist, ns

    def scan(self, hist_sum, sample_global, r2, exact):
        ex = exact or self.n_global <= self.exact_limit
        lam = r2 * sample_global / max(self.n_global, 1)
        self.guard = guard_from_hist(hist_sum, r2, lam, ex)
        cand = np.zeros_like(hist_sum)
        for q, s in enumerate(self.scores):
            e = s[s <= self.guard[q]]
            cand[q] = np.bincount(e, minlength=256)
        return cand

    def finish(self, cand_sum, r, r2):
        nq = cand_sum.shape[0]
        d = np.full((nq, r), np.inf)
        i = np.full((nq, r), -1, dtype=np.int64)
        need = np.zeros(nq, dtype=bool)
        for q in range(nq):
            B = int(self.guard[q])
            cum = np.cumsum(cand_sum[q, :B + 1])
            hit = np.flatnonzero(cum >= r2)
            if hit.size:
                bstar = int(hit[0])
            elif B >= 254:
                bstar = 254
            else:
                need[q] = True
                continue
            rows = np.flatnonzero(self.scores[q] <= bstar)
            if rows.size:
                lazy = O.LazyFull(self.cb, self.yr[q])
                dist = lazy.score(self.codes[rows])
                ids, ds = O.best_r(dist, rows + self.base, r)
                d[q, :len(ids)] = ds
                i[q, :len(ids)] = ids
        return d, i, need

    # device-protocol twins (CPU tensors): the same contract as
    # GpuShardEngine.*_dev, so shard.sharded_search_dev runs unchanged
    def context(self):
        return contextlib.nullcontext()

    def to_device(self, a):
        return torch.as_tensor(np.ascontiguousarray(a))

    torch = torch

    def begin_dev(self, y, r2, exact):
        hist, ns = self.begin(y.numpy(), r2, exact)
        return torch.as_tensor(hist.astype(np.int32)), ns

    def scan_dev(self, hist_sum, sample_global, r2, exact):
        return torch.as_tensor(self.scan(hist_sum.numpy().astype(np.int64), sample_global, r2, exact).astype(np.int32))

    def finish_dev(self, cand_sum, r, r2):
        d, i, need = self.finish(cand_sum.numpy().astype(np.int64), r, r2)
        return torch.as_tensor(d), torch.as_tensor(i), torch.as_tensor(need.astype(np.uint8))

    def merge_dev(self, parts_d, parts_i, r):
        from paper_1905_06900_b200.shard import merge_topr

        d, i = merge_topr(list(parts_d.numpy()), list(parts_i.numpy()), r)
        return torch.as_tensor(d), torch.as_tensor(i)


class ThreadComm:
    """In-process stand-in for TorchComm: shards run as threads of one
    process (one GPU) and exchange through a barrier; no kernel ever waits
    on another shard's kernel."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.slots = [None] * world
        self.local = threading.local()

    def bind(self, rank):
        self.local.rank = rank

    def _exchange(self, a):
        self.slots[self.local.rank] = a
        self.bar.wait()
        out = list(self.slots)
        self.bar.wait()
        return out

    def allreduce_sum(self, a):
        return np.sum([np.asarray(x, dtype=np.int64) for x in self._exchange(a)], axis=0)

    def allreduce_max(self, x):
        return max(self._exchange(x))

    def allgather(self, a):
        return self._exchange(a)

    # tensors (device protocol): the producing stream is drained before the
    # exchange, the result is written back in place
    def _sync(self, t):
        if t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()

    def sum_(self, t):
        self._sync(t)
        parts = self._exchange(t.clone())
        t.copy_(torch.stack(parts).sum(0).to(t.dtype))
        return t

    def max_(self, t):
        self._sync(t)
        parts = self._exchange(t.clone())
        t.copy_(torch.stack(parts).max(0).values)
        return t

    def gather_stack(self, t):
        self._sync(t)
        return torch.stack(self._exchange(t.clone()))
