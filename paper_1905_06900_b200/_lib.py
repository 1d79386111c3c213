"""ctypes binding of libdpq.so (include/dpq.h).

This is the reference-side binding a maintainer of `derivedpq` would add
(INTEGRATION.md): the reference is Python, so its FFI is ctypes over the
C ABI.  There is no CPU fallback: if the library is missing or no CUDA
device is visible, every search raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_int32, c_int64, c_uint8, c_void_p
from pathlib import Path

import numpy as np

_PATH = Path(os.environ.get("DPQ_LIB") or Path(__file__).with_name("libdpq.so"))  # DPQ_LIB: A/B another build
_lib = None

DPQ_OK, DPQ_ERR_ARG, DPQ_ERR_CUDA, DPQ_ERR_NOMEM, DPQ_ERR_STATE = 0, 1, 2, 3, 4

# name -> (restype, argtypes); mirrors include/dpq.h one-to-one
SIGNATURES = {
    "dpq_last_error": (ctypes.c_char_p, []),
    "dpq_abi_version": (c_int, []),
    "dpq_device_count": (c_int, []),
    "dpq_all_finite": (c_int, [c_void_p, c_int64]),
    "dpq_rotate_rows": (c_int, [c_void_p, c_int64, c_int64, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                                c_int]),
    "dpq_flat_create": (c_int, [c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, c_int,
                                c_int64, c_int64, c_void_p, c_int64, POINTER(c_void_p)]),
    "dpq_ivf_create": (c_int, [c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_void_p,
                               c_void_p, c_void_p, c_int, c_void_p, c_int64, POINTER(c_void_p)]),
    "dpq_destroy": (None, [c_void_p]),
    "dpq_set_stream": (c_int, [c_void_p, c_void_p]),
    "dpq_set_batch": (c_int, [c_void_p, c_int]),
    "dpq_set_check_finite": (c_int, [c_void_p, c_int]),
    "dpq_set_timing": (c_int, [c_void_p, c_int]),
    "dpq_flat_search_derived": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_int, c_void_p,
                                        c_void_p, c_void_p]),
    "dpq_flat_search_derived_dev": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p,
                                            c_void_p]),
    "dpq_flat_search_conventional": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p, c_void_p,
                                             c_void_p]),
    "dpq_ivf_probe": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p]),
    "dpq_ivf_search_derived": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_int, c_int,
                                       c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "dpq_ivf_search_conventional": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p,
                                            c_void_p, c_void_p, c_void_p, c_void_p]),
    "dpq_shard_begin": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int64, c_int, c_void_p, c_void_p]),
    "dpq_shard_scan": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int, c_int, c_void_p]),
    "dpq_shard_finish": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "dpq_shard_begin_dev": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int64, c_int, c_void_p, c_void_p]),
    "dpq_shard_scan_dev": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int, c_int, c_void_p]),
    "dpq_shard_finish_dev": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "dpq_merge_topr_dev": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int64, c_int, c_void_p, c_void_p]),
    "dpq_sync": (c_int, [c_void_p]),
    "dpq_ivf_set_shard": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64]),
    "dpq_ivf_shard_begin": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_void_p]),
    "dpq_ivf_shard_scan": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "dpq_ivf_shard_finish": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "dpq_debug_quantize_tables": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p, c_void_p,
                                          c_void_p, c_void_p]),
    "dpq_debug_low_scores": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p]),
    "dpq_debug_candidates": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p, c_void_p]),
    "dpq_debug_candidate_ids": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int64, c_void_p, c_void_p,
                                        c_void_p]),
    "dpq_debug_full_tables": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "dpq_debug_tc_tables": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "dpq_encoder_create": (c_int, [c_int, c_int, c_int, c_int, c_void_p, POINTER(c_void_p)]),
    "dpq_encoder_destroy": (None, [c_void_p]),
    "dpq_encode": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "dpq_encode_dev": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "dpq_container_read": (c_int, [c_int, ctypes.c_char_p, c_int, c_void_p, c_void_p, c_int, c_int, c_void_p,
                                   c_void_p, c_void_p]),
    "dpq_crc32_dev": (c_int, [c_int, c_void_p, c_int64, c_void_p]),
    "dpq_dev_free": (c_int, [c_int, c_void_p]),
    "dpq_dev_download": (c_int, [c_int, c_void_p, c_int64, c_void_p]),
    "dpq_dev_codes_max": (c_int, [c_int, c_void_p, c_int64, c_int, c_void_p]),
    "dpq_dev_check_permutation": (c_int, [c_int, c_void_p, c_int64, c_void_p]),
    "dpq_dev_bincount": (c_int, [c_int, c_void_p, c_int64, c_int, c_void_p, c_void_p]),
    "dpq_last_phase_ms": (c_int, [c_void_p, c_void_p]),
    "dpq_counters": (c_int, [c_void_p, c_void_p]),
    "dpq_counters_ex": (c_int, [c_void_p, c_void_p, c_int]),
}


def lib():
    """Load libdpq.so once; raise if it is absent (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not _PATH.exists():
            raise RuntimeError(
                f"{_PATH} is missing: build it with `python -m paper_1905_06900_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(str(_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    msg = lib().dpq_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == DPQ_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == DPQ_ERR_ARG:
        raise ValueError(msg)
    if rc == DPQ_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def device_count() -> int:
    return int(lib().dpq_device_count())


def require_device(device: int) -> None:
    n = device_count()
    if n <= device:
        raise RuntimeError(
            f"libdpq: CUDA device {device} not available ({n} visible); the derived search "
            "runs only on the GPU")


def ptr(a) -> c_void_p:
    """Data pointer of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return c_void_p(a.ctypes.data)
    return c_void_p(int(a.data_ptr()))


class Handle:
    """Owns one dpq_index_t*; destroyed with the Python object."""

    def __init__(self, raw: c_void_p, device: int):
        self.raw = raw
        self.device = device

    def __del__(self):
        raw = getattr(self, "raw", None)
        if raw and _lib is not None:
            _lib.dpq_destroy(raw)
            self.raw = None

    def phase_ms(self) -> np.ndarray:
        out = np.zeros(7, dtype=np.float32)
        check(lib().dpq_last_phase_ms(self.raw, ptr(out)))
        return out

    def counters(self) -> dict:
        out = np.zeros(8, dtype=np.int64)
        check(lib().dpq_counters(self.raw, ptr(out)))
        return dict(zip(("launches", "queries", "rows_scanned", "refined", "fallbacks", "emitted",
                             "table_entries", "wide_units"),
                        out.tolist()))

    def counters_ex(self) -> dict:
        out = np.zeros(12, dtype=np.int64)
        check(lib().dpq_counters_ex(self.raw, ptr(out), 12))
        return dict(zip(("launches", "queries", "rows_scanned", "refined", "fallbacks", "emitted",
                         "table_entries", "wide_units", "plane_rows", "lut_loads", "exact_reranked",
                         "probe_exact"),
                        out.tolist()))

    def set_timing(self, on: bool) -> None:
        check(lib().dpq_set_timing(self.raw, int(bool(on))))

    def set_check_finite(self, on: bool) -> None:
        check(lib().dpq_set_check_finite(self.raw, int(bool(on))))

    def set_batch(self, batch: int) -> None:
        check(lib().dpq_set_batch(self.raw, int(batch)))

    def set_stream(self, stream_ptr: int | None) -> None:
        check(lib().dpq_set_stream(self.raw, c_void_p(stream_ptr) if stream_ptr else None))


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def code_bytes_of(codes: np.ndarray) -> int:
    if codes.dtype == np.uint8:
        return 1
    if codes.dtype == np.uint16:
        return 2
    if codes.size and (codes.min() < 0 or codes.max() > 65535):
        raise ValueError("codes must fit in uint16")
    return 2 if (codes.size and codes.max() > 255) else 1


def flat_create(codebooks, derived, codes, device=0, id_base=0, prefix_codes=None) -> Handle:
    require_device(device)
    codebooks = _c(codebooks, np.float32)
    derived = _c(derived, np.float32)
    cbytes = code_bytes_of(np.asarray(codes))
    codes = _c(codes, np.uint8 if cbytes == 1 else np.uint16)
    m, k, dsub = codebooks.shape
    kbar = derived.shape[1]
    if prefix_codes is not None:
        prefix_codes = _c(prefix_codes, codes.dtype)
    out = c_void_p()
    rc = lib().dpq_flat_create(int(device), m, k, kbar, dsub, ptr(codebooks), ptr(derived), ptr(codes), cbytes,
                               int(codes.shape[0]), int(id_base), ptr(prefix_codes),
                               int(prefix_codes.shape[0]) if prefix_codes is not None else 0,
                               ctypes.byref(out))
    check(rc, "dpq_flat_create")
    return Handle(out, device)


def ivf_create(codebooks, derived, centers, offsets, sorted_codes, sorted_ids, device=0) -> Handle:
    require_device(device)
    codebooks = _c(codebooks, np.float32)
    derived = _c(derived, np.float32)
    centers = _c(centers, np.float32)
    offsets = _c(offsets, np.int64)
    cbytes = code_bytes_of(np.asarray(sorted_codes))
    sorted_codes = _c(sorted_codes, np.uint8 if cbytes == 1 else np.uint16)
    sorted_ids = _c(sorted_ids, np.int64)
    m, k, dsub = codebooks.shape
    out = c_void_p()
    rc = lib().dpq_ivf_create(int(device), m, k, derived.shape[1], dsub, ptr(codebooks), ptr(derived),
                              int(centers.shape[0]), ptr(centers), ptr(offsets), ptr(sorted_codes), cbytes,
                              ptr(sorted_ids), int(sorted_ids.shape[0]), ctypes.byref(out))
    check(rc, "dpq_ivf_create")
    return Handle(out, device)


def query_array(Y, defer_finite: bool = False):
    """Y as the reference's check_array(Y, dtype=float32, order="C") would
    return it (flat.py:71, ivf.py:125), with the common case (a 2-D,
    C-contiguous float32 ndarray) validated by one native finiteness scan
    instead of sklearn's; anything else, and every failure, goes through
    check_array itself so types and messages are the reference's.
    defer_finite: the caller's C search scans the values while it stages them
    (dpq_set_check_finite) and calls check_array itself on a failure."""
    if (isinstance(Y, np.ndarray) and type(Y) is np.ndarray and Y.ndim == 2 and Y.dtype == np.float32
            and Y.flags.c_contiguous and Y.shape[0] > 0 and Y.shape[1] > 0
            and (defer_finite or lib().dpq_all_finite(Y.ctypes.data, Y.size) == 0)):
        return Y
    from sklearn.utils.validation import check_array

    return check_array(Y, dtype=np.float32, order="C")


_CBLAS = None


def numpy_cblas():
    """(sgemv, sgemm, ilp64) entry points of the BLAS numpy links (the one
    quantizer.rotate's matmul runs on), or None when they cannot be found."""
    global _CBLAS
    if _CBLAS is None:
        import glob

        found = False
        base = Path(np.__file__).resolve().parent.parent
        for so in sorted(glob.glob(str(base / "numpy.libs" / "*openblas*.so*"))):
            try:
                B = ctypes.CDLL(so)
            except OSError:
                continue
            for pre, suf, ilp in (("scipy_cblas_", "64_", 1), ("cblas_", "64_", 1), ("scipy_cblas_", "", 0),
                                  ("cblas_", "", 0)):
                v, m = getattr(B, pre + "sgemv" + suf, None), getattr(B, pre + "sgemm" + suf, None)
                if v is not None and m is not None:
                    _CBLAS = (ctypes.cast(v, c_void_p).value, ctypes.cast(m, c_void_p).value, ilp, B)
                    found = True
                    break
            if found:
                break
        if not found:
            _CBLAS = False
    return _CBLAS or None


def _plain_rotate(quantizer) -> bool:
    """True when quantizer.rotate is `(X @ rotation_).astype(float32)` with a
    float32 (d, d) rotation (the reference's ProductQuantizer / OPQ,
    quantizer.py:235-239, and ArrayQuantizer)."""
    fn = getattr(type(quantizer), "rotate", None)
    name = (getattr(fn, "__module__", ""), getattr(fn, "__qualname__", ""))
    R = getattr(quantizer, "rotation_", None)
    return (name in {("derivedpq.quantizer", "ProductQuantizer.rotate"),
                     ("paper_1905_06900_b200.flat", "ArrayQuantizer.rotate")}
            and isinstance(R, np.ndarray) and R.dtype == np.float32 and R.ndim == 2 and R.shape[0] == R.shape[1])


def rotate_rows(quantizer, X: np.ndarray, rows_per_call: int):
    """quantizer.rotate applied to consecutive blocks of rows_per_call rows of
    X (n, d) f32, in parallel through numpy's own BLAS calls (bitwise the
    per-call results); None when that does not apply (the caller loops)."""
    blas = numpy_cblas()
    if blas is None or not _plain_rotate(quantizer):
        return None
    X = np.ascontiguousarray(X, dtype=np.float32)
    R = np.ascontiguousarray(quantizer.rotation_)
    n, d = X.shape
    if R.shape[0] != d:
        return None
    out = np.empty_like(X)
    # one host thread: OpenBLAS serialises concurrent callers behind a lock once its
    # own thread pool exists (measured ~10x slower with 2-8 callers); a plain C loop
    # of the same calls is already ~5x faster than the per-row Python loop
    check(lib().dpq_rotate_rows(ptr(X), n, int(rows_per_call), d, ptr(R), ptr(out), c_void_p(blas[0]),
                                c_void_p(blas[1]), blas[2], 1), "dpq_rotate_rows")
    # guard: the first block must equal quantizer.rotate itself (else fall back)
    g = int(rows_per_call)
    if n and not np.array_equal(out[:g].view(np.uint32),
                                np.asarray(quantizer.rotate(X[:g]), dtype=np.float32).view(np.uint32)):
        return None
    return out


class Encoder:
    """Owns one dpq_encoder_t* (tensor-core nearest-centroid encoder)."""

    def __init__(self, codebooks, device: int = 0):
        require_device(device)
        cb = _c(codebooks, np.float32)
        self.m, self.k, self.dsub = cb.shape
        self.device = device
        out = c_void_p()
        check(lib().dpq_encoder_create(int(device), self.m, self.k, self.dsub, ptr(cb), ctypes.byref(out)),
              "dpq_encoder_create")
        self.raw = out

    def __del__(self):
        raw = getattr(self, "raw", None)
        if raw and _lib is not None:
            _lib.dpq_encoder_destroy(raw)
            self.raw = None

    def encode(self, x) -> np.ndarray:
        """(n, m*dsub) f32 host -> (n, m) uint16 codes."""
        x = _c(x, np.float32)
        if x.ndim != 2 or x.shape[1] != self.m * self.dsub:
            raise ValueError(f"expected (n, {self.m * self.dsub}) input, got {x.shape}")
        out = np.empty((x.shape[0], self.m), np.uint16)
        check(lib().dpq_encode(self.raw, ptr(x), int(x.shape[0]), ptr(out)), "dpq_encode")
        return out

    def encode_dev(self, x, codes, stream_ptr: int | None = None) -> None:
        """x: CUDA tensor (n, >= m*dsub) f32 row-major; codes: CUDA int32 (n, m).
        Enqueued on `stream_ptr`, default torch's current stream of x's device
        (the legacy default stream is passed as cudaStreamLegacy, not NULL,
        which would select the encoder's private stream)."""
        import torch

        if not (isinstance(x, torch.Tensor) and isinstance(codes, torch.Tensor)):
            raise ValueError("encode_dev takes CUDA tensors")
        if x.device.type != "cuda" or x.device.index != self.device:
            raise ValueError(f"x must live on cuda:{self.device}, got {x.device}")
        if codes.device != x.device:
            raise ValueError(f"codes must live on {x.device}, got {codes.device}")
        if x.dtype != torch.float32 or x.dim() != 2 or x.stride(1) != 1 or x.shape[1] < self.m * self.dsub:
            raise ValueError(f"x must be float32 (n, >= {self.m * self.dsub}) with unit inner stride, got "
                             f"{x.dtype} {tuple(x.shape)} strides {tuple(x.stride())}")
        if codes.dtype != torch.int32 or tuple(codes.shape) != (x.shape[0], self.m) or not codes.is_contiguous():
            raise ValueError(f"codes must be a contiguous int32 ({x.shape[0]}, {self.m}) tensor, got "
                             f"{codes.dtype} {tuple(codes.shape)}")
        if stream_ptr is None:
            stream_ptr = torch.cuda.current_stream(x.device).cuda_stream
        check(lib().dpq_encode_dev(self.raw, ptr(x), int(x.shape[0]), int(x.stride(0)), ptr(codes),
                                   c_void_p(stream_ptr or 1)), "dpq_encode_dev")
