"""Shared fixtures.  `gpu` tests need a CUDA device and libdpq.so; they are
skipped (not failed) only when no device is visible at all."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and libdpq.so")


def _gpu_count() -> int:
    try:
        from paper_1905_06900_b200 import _lib
        return _lib.device_count()
    except Exception:
        return 0


def pytest_collection_modifyitems(config, items):
    if any("gpu" in it.keywords for it in items) and _gpu_count() == 0:
        skip = pytest.mark.skip(reason="no CUDA device visible")
        for it in items:
            if "gpu" in it.keywords:
                it.add_marker(skip)


def load_golden(name: str) -> dict:
    z = np.load(GOLDEN / f"{name}.npz")
    out = {k: z[k] for k in z.files}
    out["meta"] = json.loads(str(out["meta"]))
    return out


FLAT_CASES = ["pq_blobs", "pq_m2", "pq_m8", "opq_blobs"]
IVF_CASES = ["ivf_blobs", "ivf_opq"]


def c1_codebooks(g: dict) -> np.ndarray:
    """Rebuild the config-1-shape full codebooks from the seeded generator
    and the stored permutation (tests/golden/make_golden.py:c1_model)."""
    from paper_1905_06900_b200 import datagen

    seed = datagen.SEED
    st = datagen.seed_streams(seed)
    centres = datagen.sift_centres(st["centres"])
    train = datagen.sift_like(st["train"], centres, 100_000)
    pick = np.random.default_rng(seed + 7).choice(train.shape[0], size=65536, replace=False)
    temp = np.ascontiguousarray(train[pick])
    perm = g["perm"].astype(np.int64)
    return np.stack([np.ascontiguousarray(temp[:, j * 32:(j + 1) * 32])[perm[j]] for j in range(4)])


@pytest.fixture(scope="session")
def c1_golden():
    p = GOLDEN / "c1_sampled.npz"
    if not p.exists():
        pytest.skip("c1_sampled fixture not generated")
    g = load_golden("c1_sampled")
    g["codebooks"] = c1_codebooks(g)
    return g
