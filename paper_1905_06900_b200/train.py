"""GPU index-building tools for BASELINE-scale benchmarks (not the hot path).

The reference trainer/encoder need hours at 4x16 and cannot run at 10M-1B
(SURVEY §0 items 7-8, §7 step 5), so the bench builds its indexes here with
torch on the GPU:

* `train_pq`: per-subspace Lloyd k-means (seeded random init) for the
  2^b-centroid codebooks, then a balanced split into 2^bbar equal groups
  (greedy capacity assignment by assignment margin, the idea of
  clustering.py:182-203) and the re-ordering that makes the low bbar bits of
  every index its group id (quantizer.py:30-58, 190-204).  The derived
  codebooks are the group means.  The result satisfies the reference's own
  model invariant (quantizer.py:250-266).
* `encode`: nearest centroid per subspace, ties to the lowest index
  (quantizer.py:75-83 semantics; near-ties may differ from the reference's
  BLAS-dependent f32 GEMM).
* `exact_nn_gpu`: ground truth (evaluation.py:28-62): fp32 GEMM shortlist,
  f64 re-rank, ties to the lower id.
* `coarse_assign`: IVF list building in the layout of ivf.py:94-101.

These produce the SAME arrays the CPU oracle then consumes, so parity is
checked on identical inputs.
"""

from __future__ import annotations

import numpy as np
import torch


def _sqdist_argmin(x: torch.Tensor, c: torch.Tensor, c_norm: torch.Tensor, chunk: int = 8192):
    """argmin_i ||x - c_i||^2 for rows of x (fp32, TF32 allowed)."""
    out = torch.empty(x.shape[0], dtype=torch.int64, device=x.device)
    for s in range(0, x.shape[0], chunk):
        blk = x[s:s + chunk]
        d = torch.addmm(c_norm[None, :], blk, c.T, beta=1.0, alpha=-2.0)
        out[s:s + chunk] = d.argmin(dim=1)
    return out


def kmeans_gpu(x: torch.Tensor, k: int, iters: int, seed: int) -> torch.Tensor:
    g = torch.Generator(device="cpu").manual_seed(seed)
    init = torch.randperm(x.shape[0], generator=g)[:k].to(x.device)
    c = x[init].clone()
    for _ in range(iters):
        lab = _sqdist_argmin(x, c, (c * c).sum(1))
        sums = torch.zeros_like(c).index_add_(0, lab, x)
        cnt = torch.bincount(lab, minlength=k).to(x.dtype)
        nz = cnt > 0
        c[nz] = sums[nz] / cnt[nz, None]
    return c


def balanced_groups(c: torch.Tensor, kbar: int, seed: int, iters: int = 10) -> np.ndarray:
    """Equal-size partition of the k centroids into kbar groups: labels (k,)."""
    k = c.shape[0]
    if kbar == 1:
        return np.zeros(k, np.int64)
    if kbar == k:
        return np.arange(k)
    cen = kmeans_gpu(c, kbar, iters, seed)
    d2 = (torch.cdist(c.double(), cen.double()) ** 2).cpu().numpy()
    cap = k // kbar
    two = np.partition(d2, 1, axis=1)[:, :2]
    order = np.argsort(two[:, 0] - two[:, 1], kind="stable")
    ranked = np.argsort(d2, axis=1, kind="stable")
    room = np.full(kbar, cap)
    label = np.empty(k, np.int64)
    for p in order:
        row = ranked[p]
        for cc in row:
            if room[cc]:
                label[p] = cc
                room[cc] -= 1
                break
    return label


def train_pq(train: torch.Tensor, m: int, b: int, bbar: int, iters: int = 20, seed: int = 42):
    """Returns (codebooks (m,2^b,dsub) f32, derived (m,2^bbar,dsub) f32) numpy."""
    torch.backends.cuda.matmul.allow_tf32 = True
    n, d = train.shape
    dsub = d // m
    k, kbar = 1 << b, 1 << bbar
    cbs, ders = [], []
    for j in range(m):
        sub = train[:, j * dsub:(j + 1) * dsub].contiguous()
        c = kmeans_gpu(sub, k, iters, seed + j)
        label = balanced_groups(c, kbar, seed + j)
        perm = np.empty(k, np.int64)
        for gid in range(kbar):
            members = np.flatnonzero(label == gid)
            perm[(np.arange(len(members)) << bbar) | gid] = members
        cn = c.cpu().numpy()
        cbs.append(cn[perm])
        ders.append(np.stack([cn[label == gid].astype(np.float64).mean(0) for gid in range(kbar)]))
    return np.stack(cbs).astype(np.float32), np.stack(ders).astype(np.float32)


def encode(x: torch.Tensor, codebooks: np.ndarray, chunk: int = 16384) -> torch.Tensor:
    """(n, m) uint16 codes (as int32 tensor) of x on the GPU."""
    torch.backends.cuda.matmul.allow_tf32 = True
    m, k, dsub = codebooks.shape
    cb = torch.as_tensor(codebooks, device=x.device)
    out = torch.empty((x.shape[0], m), dtype=torch.int32, device=x.device)
    for j in range(m):
        c = cb[j]
        cn = (c * c).sum(1)
        sub = x[:, j * dsub:(j + 1) * dsub]
        out[:, j] = _sqdist_argmin(sub, c, cn, chunk).to(torch.int32)
    return out


def make_encoder(codebooks: np.ndarray, device=None, kind: str = "torch"):
    """x (n, m*dsub) f32 cuda tensor -> (n, m) int32 codes."""
    if kind == "torch":
        return lambda x: encode(x, codebooks)
    if kind == "tc":  # tcgen05 3xTF32 GEMM + argmin (libdpq dpq_encode_dev)
        from . import _lib

        dev = torch.device(device) if device is not None else torch.device("cuda", 0)
        enc = _lib.Encoder(codebooks, device=dev.index or 0)

        def run(x):
            x = x.contiguous()
            out = torch.empty((x.shape[0], enc.m), dtype=torch.int32, device=x.device)
            enc.encode_dev(x, out)
            return out

        run.encoder = enc
        return run
    raise ValueError(f"unknown encoder {kind!r}")


def exact_nn_gpu(db: torch.Tensor, queries: torch.Tensor, depth: int = 1, short: int = 16,
                 qchunk: int = 2048, dchunk: int = 1 << 21) -> np.ndarray:
    """Exact rank-ordered neighbours (evaluation.py:28-62 semantics)."""
    torch.backends.cuda.matmul.allow_tf32 = False
    n = db.shape[0]
    out = np.empty((queries.shape[0], depth), np.int64)
    for qs in range(0, queries.shape[0], qchunk):
        q = queries[qs:qs + qchunk]
        best_d = torch.full((q.shape[0], short), float("inf"), device=db.device)
        best_i = torch.full((q.shape[0], short), -1, dtype=torch.int64, device=db.device)
        for ds in range(0, n, dchunk):
            x = db[ds:ds + dchunk]
            d = torch.addmm((x * x).sum(1)[None, :], q, x.T, beta=1.0, alpha=-2.0)
            kk = min(short, d.shape[1])
            v, i = d.topk(kk, dim=1, largest=False)
            best_d = torch.cat([best_d, v], 1)
            best_i = torch.cat([best_i, i + ds], 1)
            v2, sel = best_d.topk(short, dim=1, largest=False)
            best_d, best_i = v2, best_i.gather(1, sel)
        # f64 re-rank of the shortlist, ties to the lower id
        cand = db[best_i.clamp_min(0)].double()
        dd = ((cand - q[:, None, :].double()) ** 2).sum(-1)
        dd[best_i < 0] = float("inf")
        dn = dd.cpu().numpy()
        ids = best_i.cpu().numpy()
        for r in range(dn.shape[0]):
            order = np.lexsort((ids[r], dn[r]))[:depth]
            out[qs + r] = ids[r][order]
    return out


def coarse_assign(x: torch.Tensor, centers: torch.Tensor) -> torch.Tensor:
    return _sqdist_argmin(x, centers, (centers * centers).sum(1))
