"""GPU drop-in for derivedpq.FlatIndex (reference flat.py:32-140).

Same constructor, fit, search signature, argument checks, exception types
and messages, result dtypes/padding and timing keys as the reference; the
search itself runs in libdpq.so on a B200.  Training and encoding are the
quantizer's own (the reference's ProductQuantizer / OPQ, or any fitted
object exposing codebooks_, derived_codebooks_, rotation_ and rotate()),
so "same encode/train outputs" holds by construction.
"""

from __future__ import annotations

import numpy as np
from sklearn.base import BaseEstimator
from sklearn.utils.validation import check_array, check_is_fitted

from . import _lib


class ArrayQuantizer:
    """A fitted quantizer assembled from arrays (the attributes the search
    reads from ProductQuantizer, quantizer.py:94-131, 235-239)."""

    def __init__(self, codebooks, derived_codebooks, rotation=None):
        self.codebooks_ = np.ascontiguousarray(codebooks, dtype=np.float32)
        self.derived_codebooks_ = np.ascontiguousarray(derived_codebooks, dtype=np.float32)
        self.rotation_ = None if rotation is None else np.ascontiguousarray(rotation, dtype=np.float32)
        self.m, self.k_, self.dsub_ = self.codebooks_.shape
        self.kbar_ = self.derived_codebooks_.shape[1]
        self.bbar_ = int(self.kbar_).bit_length() - 1
        self.b = int(self.k_ - 1).bit_length() if self.k_ > 1 else 1
        self.d_ = self.m * self.dsub_
        self.code_dtype_ = np.uint8 if self.k_ <= 256 else np.uint16

    def rotate(self, X):
        if self.rotation_ is None:
            return X
        return (X @ self.rotation_).astype(np.float32, copy=False)

    def fit(self, X, y=None):  # pragma: no cover - arrays are already fitted
        return self

    def encode(self, X) -> np.ndarray:
        """quantizer.encode (quantizer.py:165-170) on the tensor-core encoder
        (dpq_encode): rotate, nearest centroid per subspace (ties to the
        lowest index), codes in code_dtype_."""
        X = check_array(X, dtype=np.float32, order="C")
        enc = getattr(self, "_encoder", None)
        if enc is None:
            enc = self._encoder = _lib.Encoder(self.codebooks_, device=getattr(self, "device", 0))
        return enc.encode(np.ascontiguousarray(self.rotate(X), dtype=np.float32)).astype(self.code_dtype_)

    def validate(self) -> None:
        """quantizer.validate (quantizer.py:250-274): group id = low bbar
        bits of the centroid index, finite codebooks, orthonormal rotation."""
        from .errors import InvariantError

        expected = np.arange(self.k_, dtype=np.int32) & (self.kbar_ - 1)
        da = getattr(self, "derived_assignments_", None)
        if da is not None:
            for j in range(self.m):
                if not np.array_equal(da[j], expected):
                    bad = np.flatnonzero(da[j] != expected)[0]
                    raise InvariantError(f"subspace {j}: centroid {int(bad)} is in group {int(da[j][bad])}, "
                                         f"index demands {int(expected[bad])}")
        if not np.all(np.isfinite(self.codebooks_)):
            raise InvariantError("non-finite centroid in full codebooks")
        if not np.all(np.isfinite(self.derived_codebooks_)):
            raise InvariantError("non-finite centroid in derived codebooks")
        if self.rotation_ is not None:
            eye = self.rotation_.T.astype(np.float64) @ self.rotation_.astype(np.float64)
            if np.abs(eye - np.eye(self.d_)).max() > 1e-5:
                raise InvariantError("rotation matrix is not orthonormal")

    def __getstate__(self):
        state = self.__dict__.copy()
        state.pop("_encoder", None)
        return state


def rotated_queries(quantizer, Y: np.ndarray) -> np.ndarray:
    """Queries after quantizer.rotate in the reference's per-query call
    shape (1, d) (twopass.py:334): a batched (nq,d)@R differs bitwise
    from the per-row product under OpenBLAS (SURVEY Appendix A rule 11)."""
    if getattr(quantizer, "rotation_", None) is None:
        return np.ascontiguousarray(Y, dtype=np.float32)
    fast = _lib.rotate_rows(quantizer, Y, 1)  # the same BLAS call per row, on a few host threads
    if fast is not None:
        return fast
    out = np.empty((Y.shape[0], quantizer.codebooks_.shape[0] * quantizer.codebooks_.shape[2]),
                   dtype=np.float32)
    for i in range(Y.shape[0]):
        out[i] = np.asarray(quantizer.rotate(Y[i: i + 1]), dtype=np.float32).reshape(-1)
    return out


def _timings(nq: int, phase: np.ndarray | None) -> dict:
    keys = ("index_us", "tables_us", "scan_us", "refine_us")
    if phase is None:
        return {k: np.zeros(nq) for k in keys}
    return {k: np.ascontiguousarray(phase[:, i]) for i, k in enumerate(keys)}


class FlatIndex(BaseEstimator):
    """Encoded database searched on the GPU, one or two passes.

    Parameters
    ----------
    quantizer : fitted or unfitted product quantizer (reference
        ProductQuantizer / OptimizedProductQuantizer, or ArrayQuantizer).
    device : CUDA device ordinal holding the index.
    """

    def __init__(self, quantizer, device: int = 0):
        self.quantizer = quantizer
        self.device = device

    # -- build (reference flat.py:45-52, unchanged semantics) -------------
    def fit(self, X, train=None):
        X = check_array(X, dtype=np.float32, order="C")
        if not hasattr(self.quantizer, "codebooks_"):
            self.quantizer.fit(X if train is None else train)
        self.codes_ = self.quantizer.encode(X)
        self.n_ = X.shape[0]
        self._dev = None
        return self

    @classmethod
    def from_reference(cls, index, device: int = 0) -> "FlatIndex":
        """Wrap a fitted derivedpq.FlatIndex (shares its quantizer/codes)."""
        check_is_fitted(index, "codes_")
        out = cls(index.quantizer, device=device)
        out.codes_ = index.codes_
        out.n_ = index.codes_.shape[0]
        out._dev = None
        return out

    @classmethod
    def from_arrays(cls, codebooks, derived_codebooks, codes, rotation=None, device: int = 0) -> "FlatIndex":
        out = cls(ArrayQuantizer(codebooks, derived_codebooks, rotation), device=device)
        out.codes_ = np.asarray(codes)
        out.n_ = out.codes_.shape[0]
        out._dev = None
        return out

    # -- device state -----------------------------------------------------
    def _handle(self) -> _lib.Handle:
        codes = self.codes_
        key = (id(codes), codes.ctypes.data if isinstance(codes, np.ndarray) else 0, codes.shape,
               id(self.quantizer.codebooks_))
        dev = getattr(self, "_dev", None)
        if dev is None or dev[0] != key:
            h = _lib.flat_create(self.quantizer.codebooks_, self.quantizer.derived_codebooks_, codes,
                                 device=self.device)
            h.set_check_finite(True)  # host queries are validated while libdpq stages them (search below)
            self._dev = (key, h)
        return self._dev[1]

    def __getstate__(self):
        state = self.__dict__.copy()
        state.pop("_dev", None)
        return state

    # -- search (reference flat.py:54-108) ----------------------------------
    def search(self, Y, r: int, mode: str = "conventional", r2=None, capped: bool = True,
               return_timings: bool = False):
        """Top-r neighbours for each query row (see derivedpq.FlatIndex.search)."""
        check_is_fitted(self, "codes_")
        # check_array's finiteness scan (flat.py:71) rides on libdpq's staging copy of the queries
        # (dpq_set_check_finite) unless they are rotated first; it still comes before every other
        # error, as in the reference: _invalid re-runs it before raising
        # (only once the device handle exists: without a device the check must still come first)
        defer = getattr(self.quantizer, "rotation_", None) is None and getattr(self, "_dev", None) is not None
        Y = _lib.query_array(Y, defer_finite=defer)

        def _invalid(msg):
            if defer:
                from sklearn.utils.validation import check_array

                check_array(Y, dtype=np.float32, order="C")
            return ValueError(msg)

        if mode not in ("conventional", "derived"):
            raise _invalid(f"unknown mode {mode!r}")
        nq = Y.shape[0]
        if mode == "derived" and r2 is None:
            raise _invalid("derived mode requires r2")
        if nq == 0:
            dists = np.full((0, r), np.inf)
            ids = np.full((0, r), -1, dtype=np.int64)
            return (dists, ids, _timings(0, None)) if return_timings else (dists, ids)
        if mode == "derived":
            if r > r2:  # twopass.py:330-331
                raise _invalid(f"r={r} must not exceed r2={r2}")
            if self.codes_.shape[0] == 0 or r2 < 1:  # twopass.py:76-77
                raise _invalid("need at least one code to estimate qmax")
        m, _, dsub = self.quantizer.codebooks_.shape
        if Y.shape[1] != m * dsub:  # search.py:42-43
            raise _invalid(f"query dimension {Y.shape[1]} != {m}*{dsub}")
        if r < 1:  # search.py:99-101 (ResultSet)
            raise _invalid(f"result size must be >= 1, got {r}")
        yr = rotated_queries(self.quantizer, Y)
        h = self._handle()
        dists = np.empty((nq, r), dtype=np.float64)
        ids = np.empty((nq, r), dtype=np.int64)
        phase = np.zeros((nq, 4), dtype=np.float64) if return_timings else None
        L = _lib.lib()
        if mode == "derived":
            rc = L.dpq_flat_search_derived(h.raw, _lib.ptr(yr), nq, int(r), int(r2), int(bool(capped)),
                                           _lib.ptr(dists), _lib.ptr(ids), _lib.ptr(phase))
        else:
            rc = L.dpq_flat_search_conventional(h.raw, _lib.ptr(yr), nq, int(r), _lib.ptr(dists),
                                                _lib.ptr(ids), _lib.ptr(phase))
        if rc == _lib.DPQ_ERR_ARG and _lib.last_error().startswith("non-finite"):
            from sklearn.utils.validation import check_array

            check_array(Y, dtype=np.float32, order="C")  # raises the reference's ValueError
        _lib.check(rc, f"FlatIndex.search(mode={mode!r})")
        if return_timings:
            t = _timings(nq, phase)
            if mode == "conventional":
                t["refine_us"][:] = 0.0
            return dists, ids, t
        return dists, ids

    # -- unit seams (GPU twins of the reference functions the tests call) --
    def quantized_tables(self, Y, r2: int):
        """compute_tables(yr, derived) + quantize_tables(small, codes[:r2], r2)
        per query (search.py:28, twopass.py:63): (small f32 (nq,m,kbar),
        q u8 (nq,m,kbar), qmin f64 (nq,), qmax f64 (nq,))."""
        Y = check_array(Y, dtype=np.float32, order="C")
        yr = rotated_queries(self.quantizer, Y)
        nq = yr.shape[0]
        m, kbar = self.quantizer.derived_codebooks_.shape[:2]
        small = np.empty((nq, m, kbar), np.float32)
        q = np.empty((nq, m, kbar), np.uint8)
        qmin = np.empty(nq)
        qmax = np.empty(nq)
        _lib.check(_lib.lib().dpq_debug_quantize_tables(self._handle().raw, _lib.ptr(yr), nq, int(r2),
                                                        _lib.ptr(small), _lib.ptr(q), _lib.ptr(qmin),
                                                        _lib.ptr(qmax)))
        return small, q, qmin, qmax

    def candidate_counts(self, Y, r2: int):
        """b* and |candidates| per query (twopass.py:171-201, 295-302)."""
        Y = check_array(Y, dtype=np.float32, order="C")
        yr = rotated_queries(self.quantizer, Y)
        nq = yr.shape[0]
        bstar = np.empty(nq, np.int32)
        ncand = np.empty(nq, np.int64)
        _lib.check(_lib.lib().dpq_debug_candidates(self._handle().raw, _lib.ptr(yr), nq, int(r2),
                                                   _lib.ptr(bstar), _lib.ptr(ncand)))
        return bstar, ncand

    def low_scores(self, Y, r2: int):
        """adc_low_batch(codes_, quantize_tables(...)) per query
        (twopass.py:63-106): (nq, n) uint8 first-pass scores."""
        Y = check_array(Y, dtype=np.float32, order="C")
        yr = rotated_queries(self.quantizer, Y)
        out = np.empty((yr.shape[0], self.codes_.shape[0]), np.uint8)
        _lib.check(_lib.lib().dpq_debug_low_scores(self._handle().raw, _lib.ptr(yr), yr.shape[0], int(r2),
                                                   _lib.ptr(out)))
        return out

    def candidate_ids(self, Y, r2: int):
        """Per query, the ids refine scores, in the bucket-walk order of
        scan_derived + refine (twopass.py:187-217, 295-302): a list of
        (ids int64, scores uint8) pairs."""
        Y = check_array(Y, dtype=np.float32, order="C")
        yr = rotated_queries(self.quantizer, Y)
        nq = yr.shape[0]
        L, raw = _lib.lib(), self._handle().raw
        counts = np.zeros(nq, np.int64)
        _lib.check(L.dpq_debug_candidate_ids(raw, _lib.ptr(yr), nq, int(r2), 0, None, None, _lib.ptr(counts)))
        cap = int(counts.max(initial=0))
        ids = np.empty((nq, max(cap, 1)), np.int64)
        sc = np.empty((nq, max(cap, 1)), np.uint8)
        _lib.check(L.dpq_debug_candidate_ids(raw, _lib.ptr(yr), nq, int(r2), cap, _lib.ptr(ids), _lib.ptr(sc),
                                             _lib.ptr(counts)))
        return [(ids[q, :counts[q]].copy(), sc[q, :counts[q]].copy()) for q in range(nq)]

    def full_tables(self, Y):
        """compute_tables(yr, codebooks_) per query: (nq, m, k) f32."""
        Y = check_array(Y, dtype=np.float32, order="C")
        yr = rotated_queries(self.quantizer, Y)
        m, k = self.quantizer.codebooks_.shape[:2]
        out = np.empty((yr.shape[0], m, k), np.float32)
        _lib.check(_lib.lib().dpq_debug_full_tables(self._handle().raw, _lib.ptr(yr), yr.shape[0],
                                                    _lib.ptr(out)))
        return out

    def tc_tables(self, Y):
        """Tensor-core approximation of compute_tables(yr, codebooks_) with
        its error bound: (tables (nq, m, k) f32, eps (nq, m) f64)."""
        Y = check_array(Y, dtype=np.float32, order="C")
        yr = rotated_queries(self.quantizer, Y)
        m, k = self.quantizer.codebooks_.shape[:2]
        out = np.empty((yr.shape[0], m, k), np.float32)
        eps = np.empty((yr.shape[0], m), np.float64)
        _lib.check(_lib.lib().dpq_debug_tc_tables(self._handle().raw, _lib.ptr(yr), yr.shape[0], _lib.ptr(out),
                                                  _lib.ptr(eps)))
        return out, eps

    # -- persistence helpers kept from the reference (flat.py:112-126) -----
    def validate(self) -> None:
        from .errors import InvariantError

        if hasattr(self.quantizer, "validate"):
            self.quantizer.validate()
        if hasattr(self, "codes_"):
            k = self.quantizer.k_
            codes = self.codes_
            if codes.min(initial=0) < 0 or codes.max(initial=0) >= k:
                raise InvariantError(f"stored codes fall outside [0, {k})")
