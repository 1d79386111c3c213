"""Build libdpq.so (sm_100a) in-tree with nvcc.

The shared library is the product: every search the Python mirror performs
runs through it.  It is built next to this file so the snapshot that travels
to a GPU box carries it (git ignores *.so; gpurun does not).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libdpq.so"
SOURCES = ["dpq_flat.cu", "dpq_encode.cu", "dpq_tctab.cu", "dpq_container.cu"]
HEADERS = ["dpq_device.cuh", "dpq_kernels.cuh", "dpq_impl.h", "dpq_ivf.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",               # exactness: no FMA contraction anywhere
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-fopenmp",    # host staging copies on a few threads
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "dpq.h"]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False, extra=(), out: Path | None = None) -> Path:
    """Compile every source and link libdpq.so (or `out`, with `extra` nvcc
    flags: A/B variants for scripts/ab.py)."""
    lib = Path(out) if out else LIB
    if not force and not extra and out is None and not _stale():
        return LIB
    objs = []
    tmp = PKG / ("build" if not extra else "build_ab")
    tmp.mkdir(exist_ok=True)
    for src in SOURCES:
        obj = tmp / (Path(src).stem + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", str(ROOT / "include"), "-c", str(CSRC / src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}")
        (tmp / (Path(src).stem + ".ptxas.txt")).write_text(res.stderr)
        objs.append(str(obj))
    out_tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           *objs, "-o", str(out_tmp), "-lcudart", "-lgomp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("link failed")
    os.replace(out_tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
