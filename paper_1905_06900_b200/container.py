"""Model/index containers straight to the GPU.

GPU twins of derivedpq.vecio.save_model / load_model (reference
vecio.py:124-198).  The file format is the reference's, byte for byte:

    b"DPQM" | u16 version (1) | u32 header length | JSON header | arrays

with the header {"kind", "params", "arrays": [{name, dtype, shape, crc32}]}
and the raw little-endian array bytes in header order (vecio.py:131-153).

`load_model(path, verify=True, device=0)` parses the header here (it is a
few hundred bytes of JSON) and hands the bulk arrays — a flat index's
`codes`, an IVF index's `sorted_codes`, `sorted_ids` and `cell_of` — to
libdpq's `dpq_container_read`, which reads them with several host threads
into pinned buffers, copies them to HBM piece by piece, and computes their
zlib CRC-32 ON THE DEVICE.  The search handle is built from those device
buffers (no host copy of the database is ever made), and validate()'s checks
on the bulk arrays (code range, flat.py:112-118; the lists partition the
database and agree with cell_of, ivf.py:280-292) run as device reductions.
The small arrays (codebooks, rotation, centres, offsets) are read on the
host and checked with zlib exactly as the reference does.  Errors are the
reference's: FormatError for bad magic / version / header, truncated arrays
and failed checksums (same messages), InvariantError from validation;
`verify=False` skips both checks.

Bulk arrays of a loaded index stay on the device as `DeviceArray`s
(`np.asarray(index.codes_)` downloads them), so `loaded.codes_` etc. behave
as in the reference.
"""

from __future__ import annotations

import ctypes
import json
import os
import struct
import zlib

import numpy as np

from . import _lib
from .errors import FormatError, InvariantError

MAGIC = b"DPQM"
VERSION = 1
# arrays that go straight to the device, per container kind
_BULK = {"flat": ("codes",), "ivf": ("sorted_codes", "sorted_ids", "cell_of")}


class DeviceArray:
    """A device buffer owned by Python (freed with the object); np.asarray()
    downloads it."""

    def __init__(self, ptr: int, shape, dtype, device: int):
        self._ptr = int(ptr)
        self.shape = tuple(int(s) for s in shape)
        self.dtype = np.dtype(dtype)
        self.device = device
        self.ctypes = type("_ct", (), {"data": self._ptr})()  # key for the index handle caches

    @property
    def size(self) -> int:
        return int(np.prod(self.shape, dtype=np.int64))

    @property
    def nbytes(self) -> int:
        return self.size * self.dtype.itemsize

    @property
    def ndim(self) -> int:
        return len(self.shape)

    def data_ptr(self) -> int:
        return self._ptr

    def download(self) -> np.ndarray:
        out = np.empty(self.shape, dtype=self.dtype)
        _lib.check(_lib.lib().dpq_dev_download(self.device, ctypes.c_void_p(self._ptr), self.nbytes,
                                               _lib.ptr(out)), "download")
        return out

    def __array__(self, dtype=None, copy=None):
        a = self.download()
        return a if dtype is None else a.astype(dtype, copy=False)

    def __len__(self) -> int:
        return self.shape[0]

    def __del__(self):
        p = getattr(self, "_ptr", 0)
        if p and _lib._lib is not None:
            _lib._lib.dpq_dev_free(self.device, ctypes.c_void_p(p))
            self._ptr = 0

    def __repr__(self) -> str:
        return f"DeviceArray(shape={self.shape}, dtype={self.dtype}, device={self.device})"


# ------------------------------------------------------------- header --

def read_header(path):
    """(kind, params, manifest, data_start, file_size) with the reference's
    FormatError cases (vecio.py:170-181)."""
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != MAGIC:
            raise FormatError(f"{path}: bad magic {magic!r}")
        raw = f.read(6)
        if len(raw) != 6:  # struct.error in the reference; a truncated file either way
            raise FormatError(f"{path}: truncated container header")
        version, header_len = struct.unpack("<HI", raw)
        if version != VERSION:
            raise FormatError(f"{path}: unsupported container version {version}")
        try:
            header = json.loads(f.read(header_len).decode("utf-8"))
        except (UnicodeDecodeError, json.JSONDecodeError) as exc:
            raise FormatError(f"{path}: corrupt header ({exc})") from exc
    return header["kind"], header["params"], header["arrays"], 10 + header_len, size


def layout(manifest, data_start: int):
    """Byte range of every array, in header order (vecio.py:184-186)."""
    out, pos = [], data_start
    for e in manifest:
        dt = np.dtype(e["dtype"])
        shape = tuple(e["shape"])
        nb = dt.itemsize * int(np.prod(shape, dtype=np.int64))
        out.append((e["name"], dt, shape, pos, nb, e.get("crc32")))
        pos += nb
    return out


def read_arrays(path):
    """(kind, params, {name: ndarray}) read on the host without checks: for
    inspecting a container (the device loader is load_model)."""
    kind, params, manifest, start, _ = read_header(path)
    return kind, params, {name: np.fromfile(path, dtype=dt, count=int(np.prod(shape, dtype=np.int64)),
                                            offset=off).reshape(shape)
                          for name, dt, shape, off, _, _ in layout(manifest, start)}


# --------------------------------------------------------------- load --

def load_model(path, verify: bool = True, device: int = 0, threads: int | None = None):
    """GPU twin of vecio.load_model (vecio.py:156-198): a quantizer, or a
    GPU FlatIndex / IVFIndex whose bulk arrays went straight to `device`."""
    from .flat import ArrayQuantizer, FlatIndex
    from .ivf import IVFIndex

    path = str(path)
    kind, params, manifest, start, size = read_header(path)
    if kind not in ("pq", "opq", "flat", "ivf"):
        raise FormatError(f"{path}: unknown model kind {kind!r}")
    arrs = layout(manifest, start)
    for name, _, _, off, nb, _ in arrs:  # first array the file cannot hold (vecio.py:187-188)
        if off + nb > size:
            raise FormatError(f"{path}: truncated array {name!r}")
    bulk = set(_BULK.get(kind, ()))
    host, dev_idx = {}, []
    for i, (name, dt, shape, off, nb, crc) in enumerate(arrs):
        if name in bulk:
            dev_idx.append(i)
            continue
        blob = np.fromfile(path, dtype=np.uint8, count=nb, offset=off)
        host[name] = (blob, crc)
    if verify:  # host arrays first (cheap), zlib as vecio.py:189-193
        for name, (blob, crc) in host.items():
            if crc is not None and zlib.crc32(blob) != crc:
                raise FormatError(f"{path}: array {name!r} fails its checksum")
    dev = {}
    if dev_idx:
        _lib.require_device(device)
        n = len(dev_idx)
        offs = np.array([arrs[i][3] for i in dev_idx], np.int64)
        nbs = np.array([arrs[i][4] for i in dev_idx], np.int64)
        ptrs = (ctypes.c_void_p * n)()
        crcs = np.zeros(n, np.uint32)
        stats = np.zeros(4, np.float64)
        nthreads = threads or min(16, os.cpu_count() or 1)
        _lib.check(_lib.lib().dpq_container_read(int(device), path.encode(), n, _lib.ptr(offs), _lib.ptr(nbs),
                                                 int(bool(verify)), int(nthreads), ptrs, _lib.ptr(crcs),
                                                 _lib.ptr(stats)), "dpq_container_read")
        for j, i in enumerate(dev_idx):
            name, dt, shape = arrs[i][:3]
            dev[name] = (DeviceArray(ptrs[j] or 0, shape, dt, device), int(crcs[j]))
        load_model.last_stats = {"bytes": int(stats[0]), "read_s": float(stats[1]), "total_s": float(stats[2])}
    if verify:  # device-computed CRCs of the bulk arrays
        for name, _, _, _, _, crc in arrs:
            if name in dev and crc is not None and dev[name][1] != crc:
                raise FormatError(f"{path}: array {name!r} fails its checksum")
    harr = {}
    for name, dt, shape, *_ in arrs:
        if name in host:
            harr[name] = host[name][0].view(dt).reshape(shape)
    darr = {name: v[0] for name, v in dev.items()}
    if kind in ("pq", "opq"):
        model = _quantizer(kind, params, harr)
        if verify:
            model.validate()
        return model
    qarrays = {name[2:]: a for name, a in harr.items() if name.startswith("q.")}
    quant = _quantizer(params["quantizer_kind"], params["quantizer_params"], qarrays)
    if verify:
        quant.validate()
    if kind == "flat":
        codes = darr["codes"]
        idx = FlatIndex(quant, device=device)
        idx.codes_ = codes
        idx.n_ = codes.shape[0]
        if verify:
            _check_codes(codes, quant.k_, device)
        h = _flat_handle(quant, codes, device)
        idx._dev = ((id(codes), 0, codes.shape, id(quant.codebooks_)), h)
        return idx
    idx = IVFIndex(quant, n_cells=params["n_cells"], seed=params["seed"], coarse_iters=params["coarse_iters"],
                   device=device)
    idx.centers_ = np.ascontiguousarray(harr["centers"])
    idx.offsets_ = np.ascontiguousarray(harr["offsets"])
    idx.sorted_codes_ = darr["sorted_codes"]
    idx.sorted_ids_ = darr["sorted_ids"]
    idx.cell_of_ = darr["cell_of"]
    idx.n_ = idx.sorted_ids_.shape[0]
    if verify:
        _check_ivf(idx, device)
    h = _ivf_handle(quant, idx, device)
    idx._dev = ((id(idx.sorted_codes_), idx.sorted_codes_.ctypes.data, idx.sorted_codes_.shape, id(idx.centers_),
                 id(quant.codebooks_)), h)
    return idx


def _quantizer(kind, params, arrays):
    """ProductQuantizer._deserialize (quantizer.py:301-317) onto the array
    quantizer the GPU index reads."""
    from .flat import ArrayQuantizer

    q = ArrayQuantizer(arrays["codebooks"], arrays["derived_codebooks"], arrays.get("rotation"))
    q.derived_assignments_ = arrays["derived_assignments"]
    q.distortions_ = arrays["distortions"]
    q._kind = kind
    q._params = dict(params)
    q.b = int(params.get("b", q.b))
    q.code_dtype_ = np.uint8 if q.b <= 8 else np.uint16
    return q


def _check_codes(codes: DeviceArray, k: int, device: int) -> None:
    """flat.py:112-118 on the device: every stored code in [0, k)."""
    if codes.size == 0 or k >= (1 << (8 * codes.dtype.itemsize)):
        return
    mx = np.zeros(1, np.int64)
    _lib.check(_lib.lib().dpq_dev_codes_max(device, _lib.ptr(codes), codes.size, codes.dtype.itemsize,
                                            _lib.ptr(mx)), "code range")
    if mx[0] >= k:
        raise InvariantError(f"stored codes fall outside [0, {k})")


def _check_ivf(idx, device: int) -> None:
    """IVFIndex.validate (ivf.py:280-292) with the bulk checks on the device."""
    n = idx.n_
    bad = np.zeros(2, np.int64)
    if n:
        _lib.check(_lib.lib().dpq_dev_check_permutation(device, _lib.ptr(idx.sorted_ids_), n, _lib.ptr(bad)),
                   "permutation check")
    if bad.any():
        raise InvariantError("inverted lists do not partition the database")
    counts = np.zeros(idx.n_cells, np.int64)
    nbad = np.zeros(1, np.int64)
    cell = idx.cell_of_
    if isinstance(cell, DeviceArray) and cell.dtype == np.int32:  # the reference's dtype (clustering.py:64)
        _lib.check(_lib.lib().dpq_dev_bincount(device, _lib.ptr(cell), int(cell.shape[0]), int(idx.n_cells),
                                               _lib.ptr(counts), _lib.ptr(nbad)), "bincount")
    else:
        cell = np.asarray(cell)
        ok = (cell >= 0) & (cell < idx.n_cells)
        nbad[0] = int((~ok).sum())
        counts[:] = np.bincount(cell[ok], minlength=idx.n_cells)[:idx.n_cells]
    if nbad[0] or not np.array_equal(np.diff(idx.offsets_), counts):
        raise InvariantError("list offsets disagree with cell assignments")
    _check_codes(idx.sorted_codes_, idx.quantizer.k_, device)


def _flat_handle(quant, codes: DeviceArray, device: int) -> _lib.Handle:
    _lib.require_device(device)
    cb = np.ascontiguousarray(quant.codebooks_, np.float32)
    dcb = np.ascontiguousarray(quant.derived_codebooks_, np.float32)
    m, k, dsub = cb.shape
    out = ctypes.c_void_p()
    _lib.check(_lib.lib().dpq_flat_create(int(device), m, k, dcb.shape[1], dsub, _lib.ptr(cb), _lib.ptr(dcb),
                                          _lib.ptr(codes), codes.dtype.itemsize, int(codes.shape[0]), 0, None, 0,
                                          ctypes.byref(out)), "dpq_flat_create")
    return _lib.Handle(out, device)


def _ivf_handle(quant, idx, device: int) -> _lib.Handle:
    cb = np.ascontiguousarray(quant.codebooks_, np.float32)
    dcb = np.ascontiguousarray(quant.derived_codebooks_, np.float32)
    m, k, dsub = cb.shape
    centers = np.ascontiguousarray(idx.centers_, np.float32)
    offsets = np.ascontiguousarray(idx.offsets_, np.int64)
    codes = idx.sorted_codes_
    out = ctypes.c_void_p()
    _lib.check(_lib.lib().dpq_ivf_create(int(device), m, k, dcb.shape[1], dsub, _lib.ptr(cb), _lib.ptr(dcb),
                                         int(centers.shape[0]), _lib.ptr(centers), _lib.ptr(offsets),
                                         _lib.ptr(codes), codes.dtype.itemsize, _lib.ptr(idx.sorted_ids_),
                                         int(idx.n_), ctypes.byref(out)), "dpq_ivf_create")
    return _lib.Handle(out, device)


# --------------------------------------------------------------- save --

def serialize(model):
    """(kind, params, arrays) as the reference's _serialize methods
    (quantizer.py:289-299, flat.py:120-126, ivf.py:297-316)."""
    from sklearn.utils.validation import check_is_fitted

    if hasattr(model, "_serialize") and not _is_mirror(model):
        return model._serialize()
    if hasattr(model, "codebooks_"):  # a quantizer (ArrayQuantizer from load_model)
        arrays = {"codebooks": model.codebooks_, "derived_codebooks": model.derived_codebooks_,
                  "derived_assignments": getattr(model, "derived_assignments_", None),
                  "distortions": getattr(model, "distortions_", None)}
        if arrays["derived_assignments"] is None:  # the index invariant (quantizer.py:258)
            arrays["derived_assignments"] = np.tile(np.arange(model.k_, dtype=np.int32) & (model.kbar_ - 1),
                                                    (model.m, 1))
        if arrays["distortions"] is None:
            raise ValueError("quantizer has no distortions_; cannot write a reference container")
        if getattr(model, "rotation_", None) is not None:
            arrays["rotation"] = model.rotation_
        kind = getattr(model, "_kind", "opq" if getattr(model, "rotation_", None) is not None else "pq")
        params = getattr(model, "_params", None)
        if params is None:
            raise ValueError("quantizer has no training parameters; cannot write a reference container")
        return kind, params, arrays
    from .flat import FlatIndex
    from .ivf import IVFIndex

    qkind, qparams, qarrays = serialize(model.quantizer)
    if isinstance(model, FlatIndex):
        check_is_fitted(model, "codes_")
        arrays = {"codes": np.asarray(model.codes_)}
        arrays.update({f"q.{k}": v for k, v in qarrays.items()})
        return "flat", {"quantizer_kind": qkind, "quantizer_params": qparams}, arrays
    if isinstance(model, IVFIndex):
        check_is_fitted(model, "centers_")
        params = {"n_cells": model.n_cells, "seed": model.seed, "coarse_iters": model.coarse_iters,
                  "quantizer_kind": qkind, "quantizer_params": qparams}
        arrays = {"centers": model.centers_, "cell_of": np.asarray(model.cell_of_),
                  "sorted_ids": np.asarray(model.sorted_ids_), "sorted_codes": np.asarray(model.sorted_codes_),
                  "offsets": model.offsets_}
        arrays.update({f"q.{k}": v for k, v in qarrays.items()})
        return "ivf", params, arrays
    raise TypeError(f"cannot serialize {type(model).__name__}")


def _is_mirror(model) -> bool:
    return type(model).__module__.startswith(__package__ or "paper_1905_06900_b200")


def save_model(model, path) -> None:
    """vecio.save_model (vecio.py:124-153): the same bytes the reference
    writes for the same arrays."""
    kind, params, arrays = serialize(model)
    manifest, blobs = [], []
    for name, arr in arrays.items():
        arr = np.ascontiguousarray(arr)
        blob = arr.tobytes()
        manifest.append({"name": name, "dtype": arr.dtype.str, "shape": list(arr.shape),
                         "crc32": zlib.crc32(blob)})
        blobs.append(blob)
    header = json.dumps({"kind": kind, "params": params, "arrays": manifest}).encode("utf-8")
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<HI", VERSION, len(header)))
        f.write(header)
        for blob in blobs:
            f.write(blob)


def crc32_device(buf, device: int = 0) -> int:
    """zlib.crc32 of a device buffer (torch tensor or DeviceArray), on the
    device."""
    out = np.zeros(1, np.uint32)
    n = buf.nbytes if hasattr(buf, "nbytes") and isinstance(buf, DeviceArray) else buf.numel() * buf.element_size()
    _lib.check(_lib.lib().dpq_crc32_dev(int(device), _lib.ptr(buf), int(n), _lib.ptr(out)), "dpq_crc32_dev")
    return int(out[0])


__all__ = ["load_model", "save_model", "DeviceArray", "read_header", "read_arrays", "layout", "crc32_device"]
