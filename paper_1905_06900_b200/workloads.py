"""BASELINE.json workloads for bench.py and the full-size parity runs
(benchmark tooling, not the search path).

Each config is a seeded synthetic stand-in of BASELINE.json's configs
(SIFT1M/1B and GIST are not available): codebooks trained on
the GPU (train.py), database rows generated on the GPU in fixed global
chunks of 2^20 rows (so any row range — a shard — is reproducible without
generating the rest), encoded with the tensor-core encoder, and exact
rank-0 ground truth (evaluation.py:28-62 semantics) accumulated chunk by
chunk.

  c2  configs[1]: flat PQ 4x16 + derived 4x8, SIFT-like, N = 10M, r2 = 1000
  c3  configs[2]: OPQ 4x16 + derived 4x8 — the data are rotated by a seeded
      orthogonal matrix R0 and the quantizer's rotation is R0^T (it undoes
      it exactly instead of being learned), N = 100M, r2 = 2000
  c5  configs[4]: flat PQ 8x16 + derived 8x8, 960-d GIST-like, dsub = 120,
      N = 50M, r2 = 2000, 4096-query batches
"""

from __future__ import annotations

import numpy as np

from . import datagen

CHUNK = 1 << 20  # global generation chunk (rows)

CONFIGS = {
    "c2": dict(name="c2", kind="flat", m=4, dsub=32, n=10_000_000, r2=1000, r=100, batch=1024, data="sift",
               opq=False, baseline="configs[1]",
               label="BASELINE configs[1]: flat PQ 4x16 + derived 4x8, SIFT-like, N=10M, 1024-query batches, "
                     "r2=1000, k=100"),
    "c3": dict(name="c3", kind="flat", m=4, dsub=32, n=100_000_000, r2=2000, r=100, batch=1024, data="sift",
               opq=True, baseline="configs[2]",
               label="BASELINE configs[2]: OPQ 4x16 + derived 4x8, SIFT-like rotated by a seeded orthogonal "
                     "matrix, N=100M sharded evenly over the GPUs, 1024-query batches, r2=2000, k=100"),
    "c5": dict(name="c5", kind="flat", m=8, dsub=120, n=50_000_000, r2=2000, r=100, batch=4096, data="gist",
               opq=False, baseline="configs[4]",
               label="BASELINE configs[4]: flat PQ 8x16 + derived 8x8, GIST-like 960-d, N=50M, 4096-query "
                     "batches, r2=2000, k=100"),
}


def dim(cfg) -> int:
    return cfg["m"] * cfg["dsub"]


def centres_of(cfg, seed: int):
    st = datagen.seed_streams(seed)
    if cfg["data"] == "sift":
        return datagen.sift_centres(st["centres"]), st
    return datagen.gist_centres(st["centres"]), st


def data_rotation(cfg, seed: int):
    """R0 (data frame) for OPQ configs, else None."""
    return datagen.random_orthogonal(dim(cfg), seed + 3) if cfg["opq"] else None


def gen_chunk(cfg, centres_t, seed: int, ci: int, device):
    """Global chunk ci: rows [ci * CHUNK, min(n, (ci+1) * CHUNK)) (torch Philox
    seeded by (seed, ci)), in the raw (unrotated) frame."""
    import torch

    n = cfg["n"]
    s, e = ci * CHUNK, min(n, (ci + 1) * CHUNK)
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1_000_003 + ci)
    pick = torch.randint(0, centres_t.shape[0], (e - s,), generator=g, device=device)
    noise = torch.randn((e - s, centres_t.shape[1]), generator=g, device=device)
    if cfg["data"] == "sift":
        return (centres_t[pick] + noise.abs_().mul_(20.0)).round_().clamp_(0, 255)
    return (centres_t[pick] + noise.mul_(0.05)).clamp_(0.0, 1.0)


def row_chunks(cfg, centres, seed: int, lo: int, hi: int, device):
    """Yields (row0, x) for the database rows [lo, hi) in the DATA frame
    (rotated by R0 for OPQ configs), chunk by chunk."""
    import torch

    ct = torch.as_tensor(np.asarray(centres), dtype=torch.float32, device=device)
    R0 = data_rotation(cfg, seed)
    R0t = torch.as_tensor(R0, device=device) if R0 is not None else None
    for ci in range(lo // CHUNK, (hi + CHUNK - 1) // CHUNK):
        s = ci * CHUNK
        x = gen_chunk(cfg, ct, seed + 1, ci, device)
        a, b = max(lo, s) - s, min(hi, s + x.shape[0]) - s
        x = x[a:b]
        if R0t is not None:
            x = x @ R0t
        yield s + a, x


def train_model(cfg, seed: int, device, train_n: int = 100_000, iters: int = 12):
    """(codebooks, derived, rotation): rotation = R0^T for OPQ configs (the
    quantizer rotates queries/data back into the frame it was trained in)."""
    import torch

    from . import train

    centres, st = centres_of(cfg, seed)
    tr = datagen.sift_like(st["train"], centres, train_n) if cfg["data"] == "sift" else \
        datagen.gist_like(st["train"], centres, train_n)
    trt = torch.as_tensor(tr, device=device)
    cb, der = train.train_pq(trt, cfg["m"], 16, 8, iters=iters, seed=seed)
    R0 = data_rotation(cfg, seed)
    rot = None if R0 is None else np.ascontiguousarray(R0.T)
    return cb, der, rot


def queries(cfg, seed: int, nq: int) -> np.ndarray:
    """nq seeded queries in the data frame (numpy, f32)."""
    centres, st = centres_of(cfg, seed)
    Y = datagen.sift_like(st["queries"], centres, nq) if cfg["data"] == "sift" else \
        datagen.gist_like(st["queries"], centres, nq)
    R0 = data_rotation(cfg, seed)
    return Y if R0 is None else (Y @ R0).astype(np.float32)


class StreamingTruth:
    """Exact rank-0 nearest neighbour of each query over streamed database
    chunks (evaluation.py:28-62: f64 distances, ties to the lower id): an
    fp32 GEMM shortlist of `short` rows per query, re-ranked in f64."""

    def __init__(self, Y, device, short: int = 16):
        import torch

        self.torch = torch
        self.q = torch.as_tensor(np.asarray(Y, np.float32), device=device)
        nq, d = self.q.shape
        self.short = short
        self.bd = torch.full((nq, short), float("inf"), device=device)
        self.bi = torch.full((nq, short), -1, dtype=torch.int64, device=device)
        self.bv = torch.zeros((nq, short, d), device=device)

    def update(self, row0: int, x):
        torch = self.torch
        torch.backends.cuda.matmul.allow_tf32 = False
        qn = (self.q * self.q).sum(1)
        for qs in range(0, self.q.shape[0], 4096):
            q = self.q[qs:qs + 4096]
            d = torch.addmm((x * x).sum(1)[None, :], q, x.T, beta=1.0, alpha=-2.0) + qn[qs:qs + 4096, None]
            kk = min(self.short, d.shape[1])
            v, i = d.topk(kk, dim=1, largest=False)
            cd = torch.cat([self.bd[qs:qs + 4096], v], 1)
            ci = torch.cat([self.bi[qs:qs + 4096], i + row0], 1)
            cv = torch.cat([self.bv[qs:qs + 4096], x[i]], 1)
            v2, sel = cd.topk(self.short, dim=1, largest=False)
            self.bd[qs:qs + 4096] = v2
            self.bi[qs:qs + 4096] = ci.gather(1, sel)
            self.bv[qs:qs + 4096] = cv.gather(1, sel[:, :, None].expand(-1, -1, cv.shape[2]))

    def result(self):
        """(d64 (nq,), id (nq,)): the best (distance, id) pair per query."""
        dd = ((self.bv.double() - self.q[:, None, :].double()) ** 2).sum(-1)
        dd[self.bi < 0] = float("inf")
        dn, ids = dd.cpu().numpy(), self.bi.cpu().numpy()
        out_d = np.empty(dn.shape[0])
        out_i = np.empty(dn.shape[0], np.int64)
        for r in range(dn.shape[0]):
            o = np.lexsort((ids[r], dn[r]))[0]
            out_d[r], out_i[r] = dn[r, o], ids[r, o]
        return out_d, out_i


def merge_truth(parts):
    """Global rank-0 neighbour from per-shard (d64, id) results: the
    lexicographic (distance, id) minimum."""
    d = np.stack([p[0] for p in parts], 1)
    i = np.stack([p[1] for p in parts], 1)
    out = np.empty(d.shape[0], np.int64)
    for r in range(d.shape[0]):
        out[r] = i[r, np.lexsort((i[r], d[r]))[0]]
    return out


def encode_rows(cfg, codebooks, rotation, centres, seed: int, lo: int, hi: int, device, truth=None,
                encoder: str = "tc"):
    """Codes (hi - lo, m) uint16 of database rows [lo, hi); the rows also
    stream through `truth` (StreamingTruth) when given."""
    import torch

    from . import train

    enc = train.make_encoder(codebooks, device=device, kind=encoder if cfg["dsub"] <= 128 else "torch")
    rot_t = torch.as_tensor(rotation, device=device) if rotation is not None else None
    codes = np.empty((hi - lo, cfg["m"]), np.uint16)
    for row0, x in row_chunks(cfg, centres, seed, lo, hi, device):
        if truth is not None:
            truth.update(row0, x)
        xe = x @ rot_t if rot_t is not None else x  # quantizer.rotate of the data (encode, quantizer.py:208-214)
        codes[row0 - lo:row0 - lo + x.shape[0]] = enc(xe).cpu().numpy().astype(np.uint16)
    return codes
