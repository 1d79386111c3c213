"""GPU drop-in for derivedpq.IVFIndex (reference ivf.py:178-340).

Same constructor parameters, probe/search signatures, argument checks,
exception types, result conventions and timing keys as the reference; probe
and search run in libdpq.so.  Training (coarse k-means, residual PQ) is the
reference's: `fit` delegates to derivedpq when it is importable, otherwise
build the index offline and wrap it with `from_reference` / `from_arrays`.
"""

from __future__ import annotations

import numpy as np
from sklearn.base import BaseEstimator
from sklearn.utils.validation import check_array, check_is_fitted

from . import _lib
from .flat import ArrayQuantizer, _timings


class IVFIndex(BaseEstimator):
    """Inverted file over residual product-quantizer codes, searched on GPU."""

    def __init__(self, quantizer, n_cells: int = 256, seed: int = 42, coarse_iters: int = 50, device: int = 0):
        self.quantizer = quantizer
        self.n_cells = n_cells
        self.seed = seed
        self.coarse_iters = coarse_iters
        self.device = device

    # -- build ------------------------------------------------------------
    def fit(self, X, train=None):
        """ivf.py:63-103, by the reference trainer (offline, not the hot path)."""
        try:
            from derivedpq import IVFIndex as _RefIVF
        except ImportError as exc:  # pragma: no cover - depends on the host
            raise ImportError(
                "IVFIndex.fit trains with the reference package derivedpq; build the index with it "
                "and wrap it via IVFIndex.from_reference(...)") from exc
        ref = _RefIVF(self.quantizer, n_cells=self.n_cells, seed=self.seed,
                      coarse_iters=self.coarse_iters).fit(X, train)
        self._adopt(ref)
        return self

    def _adopt(self, ref):
        self.quantizer = ref.quantizer
        self.centers_ = ref.centers_
        self.cell_of_ = ref.cell_of_
        self.sorted_ids_ = ref.sorted_ids_
        self.sorted_codes_ = ref.sorted_codes_
        self.offsets_ = ref.offsets_
        self.row_of_ = ref.row_of_
        self.n_ = ref.n_
        self._dev = None

    @classmethod
    def from_reference(cls, index, device: int = 0) -> "IVFIndex":
        check_is_fitted(index, "centers_")
        out = cls(index.quantizer, n_cells=index.n_cells, seed=index.seed, coarse_iters=index.coarse_iters,
                  device=device)
        out._adopt(index)
        return out

    @classmethod
    def from_arrays(cls, codebooks, derived_codebooks, centers, offsets, sorted_codes, sorted_ids,
                    cell_of=None, rotation=None, device: int = 0) -> "IVFIndex":
        centers = np.ascontiguousarray(centers, dtype=np.float32)
        out = cls(ArrayQuantizer(codebooks, derived_codebooks, rotation), n_cells=centers.shape[0], device=device)
        out.centers_ = centers
        out.offsets_ = np.ascontiguousarray(offsets, dtype=np.int64)
        out.sorted_codes_ = np.asarray(sorted_codes)
        out.sorted_ids_ = np.ascontiguousarray(sorted_ids, dtype=np.int64)
        n = out.sorted_ids_.shape[0]
        out.n_ = n
        out.row_of_ = np.empty(n, dtype=np.int64)
        out.row_of_[out.sorted_ids_] = np.arange(n)
        if cell_of is None:
            cell_of = np.repeat(np.arange(centers.shape[0]), np.diff(out.offsets_))[out.row_of_]
        out.cell_of_ = np.asarray(cell_of)
        out._dev = None
        return out

    def _handle(self) -> _lib.Handle:
        key = (id(self.sorted_codes_), self.sorted_codes_.ctypes.data, self.sorted_codes_.shape,
               id(self.centers_), id(self.quantizer.codebooks_))
        dev = getattr(self, "_dev", None)
        if dev is None or dev[0] != key:
            h = _lib.ivf_create(self.quantizer.codebooks_, self.quantizer.derived_codebooks_, self.centers_,
                                self.offsets_, self.sorted_codes_, self.sorted_ids_, device=self.device)
            self._dev = (key, h)
        return self._dev[1]

    def __getstate__(self):
        state = self.__dict__.copy()
        state.pop("_dev", None)
        return state

    # -- query ------------------------------------------------------------
    def _probe_cells(self, Y: np.ndarray, ma: int) -> np.ndarray:
        cells = np.empty((Y.shape[0], ma), dtype=np.int64)
        if Y.shape[0]:
            _lib.check(_lib.lib().dpq_ivf_probe(self._handle().raw, _lib.ptr(Y), Y.shape[0], int(ma),
                                                _lib.ptr(cells)), "IVFIndex.probe")
        return cells

    def probe(self, y, ma: int):
        """ivf.py:107-120: (cells ascending by centre distance, residuals)."""
        check_is_fitted(self, "centers_")
        y = np.asarray(y, dtype=np.float32).reshape(-1)
        if not (1 <= ma <= self.n_cells):
            raise ValueError(f"ma must be in [1, {self.n_cells}], got {ma}")
        cells = self._probe_cells(np.ascontiguousarray(y[None, :]), ma)[0]
        return cells, y[None, :] - self.centers_[cells]

    def search(self, Y, r: int, ma: int = 8, mode: str = "conventional", r2=None, capped: bool = True,
               return_timings: bool = False):
        """Top-r neighbours of each query over the ma nearest cells
        (see derivedpq.IVFIndex.search, ivf.py:125-160)."""
        check_is_fitted(self, "centers_")
        Y = _lib.query_array(Y)
        if mode not in ("conventional", "derived"):
            raise ValueError(f"unknown mode {mode!r}")
        if mode == "derived":
            if r2 is None:
                raise ValueError("derived mode requires r2")
            if r > r2:
                raise ValueError(f"r={r} must not exceed r2={r2}")
        nq = Y.shape[0]
        if nq == 0:
            d, i = np.full((0, r), np.inf), np.full((0, r), -1, dtype=np.int64)
            return (d, i, _timings(0, None)) if return_timings else (d, i)
        if not (1 <= ma <= self.n_cells):  # ivf.py:115-116 (first query's probe)
            raise ValueError(f"ma must be in [1, {self.n_cells}], got {ma}")
        if Y.shape[1] != self.centers_.shape[1]:  # ivf.py:117 broadcasting error
            raise ValueError(f"query dimension {Y.shape[1]} != {self.centers_.shape[1]}")
        if r < 1:
            raise ValueError(f"result size must be >= 1, got {r}")
        h = self._handle()
        res_rot = cells = None
        if getattr(self.quantizer, "rotation_", None) is not None:
            # OPQ: residuals rotated by the reference's own rotate in its
            # (ma, d) call shape (ivf.py:202), so tables are bitwise its own
            cells = self._probe_cells(Y, ma)
            res = (Y[:, None, :] - self.centers_[cells]).reshape(nq * ma, Y.shape[1])  # ivf.py:120, f32
            fast = _lib.rotate_rows(self.quantizer, res, ma)  # the same BLAS call per query, threaded
            if fast is not None:
                res_rot = fast.reshape(nq, ma, Y.shape[1])
            else:
                res_rot = np.empty((nq, ma, Y.shape[1]), dtype=np.float32)
                for qi in range(nq):
                    res_q = Y[qi][None, :] - self.centers_[cells[qi]]
                    res_rot[qi] = np.asarray(self.quantizer.rotate(res_q), dtype=np.float32)
        dists = np.empty((nq, r), dtype=np.float64)
        ids = np.empty((nq, r), dtype=np.int64)
        phase = np.zeros((nq, 4), dtype=np.float64) if return_timings else None
        L = _lib.lib()
        if mode == "derived":
            rc = L.dpq_ivf_search_derived(h.raw, _lib.ptr(Y), nq, int(r), int(ma), int(r2), int(bool(capped)),
                                          _lib.ptr(res_rot), _lib.ptr(cells), _lib.ptr(dists), _lib.ptr(ids),
                                          _lib.ptr(phase))
        else:
            rc = L.dpq_ivf_search_conventional(h.raw, _lib.ptr(Y), nq, int(r), int(ma), _lib.ptr(res_rot),
                                               _lib.ptr(cells), _lib.ptr(dists), _lib.ptr(ids), _lib.ptr(phase))
        _lib.check(rc, f"IVFIndex.search(mode={mode!r})")
        if return_timings:
            t = _timings(nq, phase)
            if mode == "conventional":
                t["refine_us"][:] = 0.0
            return dists, ids, t
        return dists, ids

    def validate(self) -> None:
        from .errors import InvariantError

        check_is_fitted(self, "centers_")
        if hasattr(self.quantizer, "validate"):
            self.quantizer.validate()
        if not np.array_equal(np.sort(self.sorted_ids_), np.arange(self.n_)):
            raise InvariantError("inverted lists do not partition the database")
        codes = self.sorted_codes_
        k = self.quantizer.k_
        if codes.min(initial=0) < 0 or codes.max(initial=0) >= k:
            raise InvariantError(f"stored codes fall outside [0, {k})")
