"""Seeded synthetic data of BASELINE.json's shapes (stand-ins for SIFT/GIST).

SIFT1M/SIFT1B/TINY10M are not available, so the benchmark and
the parity suites use:

* SIFT-like (configs 1-4): 256 mixture centres uniform in [0, 64]^128, each
  vector = a random centre + |N(0, 20)| per dimension, rounded and clipped
  to [0, 255], float32.
* GIST-like (config 5): 512 centres uniform in [0, 1]^960, + N(0, 0.05),
  clipped to [0, 1].

CPU generation (numpy, PCG64) is used for anything the CPU oracle or the
reference must also see; GPU generation (torch Philox, chunked) for the
10M-1B databases the bench needs.  Both are deterministic per seed; they
do not produce the same numbers as each other and do not need to.
"""

from __future__ import annotations

import numpy as np

SEED = 42  # the reference CLI default (cli.py:235)
STREAMS = ("centres", "train", "database", "queries")


def seed_streams(seed: int = SEED):
    """np.random.SeedSequence(seed).spawn(4) -> generators for the four
    roles in STREAMS (SURVEY §8d seeding proposal)."""
    kids = np.random.SeedSequence(seed).spawn(len(STREAMS))
    return {name: np.random.default_rng(k) for name, k in zip(STREAMS, kids)}


def sift_centres(rng: np.random.Generator, n_centres: int = 256, d: int = 128) -> np.ndarray:
    return rng.uniform(0.0, 64.0, size=(n_centres, d))


def sift_like(rng: np.random.Generator, centres: np.ndarray, n: int, chunk: int = 1 << 18) -> np.ndarray:
    """n SIFT-like float32 vectors drawn around `centres` (numpy)."""
    d = centres.shape[1]
    out = np.empty((n, d), dtype=np.float32)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        pick = rng.integers(centres.shape[0], size=e - s)
        x = centres[pick] + np.abs(rng.normal(0.0, 20.0, size=(e - s, d)))
        out[s:e] = np.clip(np.rint(x), 0, 255)
    return out


def gist_centres(rng: np.random.Generator, n_centres: int = 512, d: int = 960) -> np.ndarray:
    return rng.uniform(0.0, 1.0, size=(n_centres, d))


def gist_like(rng: np.random.Generator, centres: np.ndarray, n: int, chunk: int = 1 << 16) -> np.ndarray:
    d = centres.shape[1]
    out = np.empty((n, d), dtype=np.float32)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        pick = rng.integers(centres.shape[0], size=e - s)
        out[s:e] = np.clip(centres[pick] + rng.normal(0.0, 0.05, size=(e - s, d)), 0.0, 1.0)
    return out


def gaussian_blobs(n, d, n_blobs, seed, spread=0.05, box=1.0):
    """Clustered data of the reference's own test fixture shape
    (tests/conftest.py:5-11 of the reference), restated."""
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-box, box, size=(n_blobs, d))
    assign = rng.integers(n_blobs, size=n)
    return (centers[assign] + rng.normal(0.0, spread, size=(n, d))).astype(np.float32)


def random_orthogonal(d: int, seed: int) -> np.ndarray:
    """Seeded random orthogonal matrix (QR of a normal matrix), float32 —
    config 3's data rotation."""
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.normal(size=(d, d)))
    q = q * np.sign(np.diag(r))[None, :]
    return q.astype(np.float32)


# ------------------------------------------------------------------ GPU --

def sift_like_torch(n: int, seed: int, centres, device="cuda", chunk: int = 1 << 22, out=None):
    """n SIFT-like vectors generated on the GPU in seeded chunks.

    centres: (256, 128) array (numpy or torch).  Chunk c uses a torch
    generator seeded with (seed, c) so any prefix of the database is
    reproducible without generating the rest."""
    import torch

    c = torch.as_tensor(np.asarray(centres), dtype=torch.float32, device=device)
    d = c.shape[1]
    if out is None:
        out = torch.empty((n, d), dtype=torch.float32, device=device)
    g = torch.Generator(device=device)
    for ci, s in enumerate(range(0, n, chunk)):
        e = min(n, s + chunk)
        g.manual_seed(seed * 1_000_003 + ci)
        pick = torch.randint(0, c.shape[0], (e - s,), generator=g, device=device)
        x = c[pick] + torch.randn((e - s, d), generator=g, device=device).abs_().mul_(20.0)
        out[s:e] = x.round_().clamp_(0, 255)
    return out
