"""Model containers straight to the device on the GPU:
dpq_crc32_dev == zlib.crc32, containers written by the REFERENCE
(tests/golden/containers) load through dpq_container_read and search
bit-identically to the reference's own results, device validation raises the
reference's errors, and a BASELINE-shape flat index (PQ 4x16, 2M codes)
round-trips save_model -> load_model."""

from __future__ import annotations

import json
import zlib
from pathlib import Path

import numpy as np
import pytest

from paper_1905_06900_b200 import FormatError, InvariantError
from paper_1905_06900_b200 import container as C
from paper_1905_06900_b200.flat import FlatIndex
from paper_1905_06900_b200.ivf import IVFIndex

pytestmark = pytest.mark.gpu
FIX = Path(__file__).resolve().parent / "golden" / "containers"


def _fix(case):
    z = np.load(FIX / f"{case}.npz")
    out = {k: z[k] for k in z.files}
    if "meta" in out:
        out["meta"] = json.loads(str(out["meta"]))
    return out


@pytest.mark.parametrize("n", [0, 1, 5, 16, 4095, 262144, 262144 + 7, 3 * 262144 + 4100, (40 << 20) + 13])
def test_device_crc32_equals_zlib(n):
    import torch

    data = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8)
    t = torch.as_tensor(data).cuda()
    assert C.crc32_device(t) == zlib.crc32(data.tobytes())


def test_device_crc32_rejects_unaligned():
    import torch

    t = torch.zeros(1024, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="aligned"):
        C.crc32_device(t[3:])


@pytest.mark.parametrize("case", ["flat_u8", "flat_u16", "flat_opq"])
def test_reference_flat_container_searches_like_the_reference(case):
    g = _fix(case)
    idx = C.load_model(FIX / f"{case}.dpq")
    assert isinstance(idx, FlatIndex) and isinstance(idx.codes_, C.DeviceArray)
    _, _, arrays = C.read_arrays(FIX / f"{case}.dpq")
    np.testing.assert_array_equal(np.asarray(idx.codes_), arrays["codes"])
    m = g["meta"]
    d, i = idx.search(g["queries"], m["r"], mode="derived", r2=m["r2"])
    np.testing.assert_array_equal(i, g["exp_der_i"])
    np.testing.assert_array_equal(d, g["exp_der_d"])
    if "exp_conv_i" in g:
        d, i = idx.search(g["queries"], m["r"])
        np.testing.assert_array_equal(i, g["exp_conv_i"])
        np.testing.assert_array_equal(d, g["exp_conv_d"])


def test_reference_ivf_container_searches_like_the_reference(tmp_path):
    g = _fix("ivf_small")
    idx = C.load_model(FIX / "ivf_small.dpq")
    assert isinstance(idx, IVFIndex)
    m = g["meta"]
    d, i = idx.search(g["queries"], m["r"], ma=m["ma"], mode="derived", r2=m["r2"])
    np.testing.assert_array_equal(i, g["exp_der_i"])
    np.testing.assert_array_equal(d, g["exp_der_d"])
    d, i = idx.search(g["queries"], m["r"], ma=m["ma"])
    np.testing.assert_array_equal(i, g["exp_conv_i"])
    np.testing.assert_array_equal(d, g["exp_conv_d"])
    out = tmp_path / "again.dpq"  # device arrays download for save_model: same bytes
    C.save_model(idx, out)
    assert out.read_bytes() == (FIX / "ivf_small.dpq").read_bytes()


def test_loaded_flat_round_trips_byte_identically(tmp_path):
    idx = C.load_model(FIX / "flat_u16.dpq")
    out = tmp_path / "again.dpq"
    C.save_model(idx, out)
    assert out.read_bytes() == (FIX / "flat_u16.dpq").read_bytes()


def test_quantizer_encodes_like_the_reference():
    q = C.load_model(FIX / "pq_small.dpq")
    g = _fix("pq_small")
    codes = q.encode(g["X"])
    assert codes.dtype == g["codes"].dtype
    assert np.mean(codes == g["codes"]) > 0.995  # f32 near-ties only (the reference's BLAS GEMM)


def _flip(tmp_path, case, name, byte_in_array=5):
    path = FIX / f"{case}.dpq"
    _, _, manifest, start, _ = C.read_header(path)
    off = [a for a in C.layout(manifest, start) if a[0] == name][0][3]
    blob = bytearray(path.read_bytes())
    blob[off + byte_in_array] ^= 0x5A
    p = tmp_path / f"flip_{name}.dpq"
    p.write_bytes(bytes(blob))
    return p


@pytest.mark.parametrize("case,name", [("flat_u8", "codes"), ("ivf_small", "sorted_codes"),
                                       ("ivf_small", "sorted_ids"), ("ivf_small", "cell_of")])
def test_device_checksum_catches_flipped_bulk_byte(tmp_path, case, name):
    p = _flip(tmp_path, case, name)
    with pytest.raises(FormatError, match=f"array '{name}' fails its checksum"):
        C.load_model(p)
    C.load_model(p, verify=False)  # no checksum, no validation


def test_device_validation_code_range(tmp_path):
    kind, params, arrays = C.read_arrays(FIX / "flat_u16.dpq")
    k = arrays["q.codebooks"].shape[1]
    codes = arrays["codes"].copy()
    codes[123, 1] = k  # out of [0, k) with a correct checksum
    idx = C.load_model(FIX / "flat_u16.dpq")
    idx.codes_ = codes
    p = tmp_path / "range.dpq"
    C.save_model(idx, p)
    with pytest.raises(InvariantError, match=r"stored codes fall outside \[0, 1024\)"):
        C.load_model(p)


def test_device_validation_ivf_partition_and_cells(tmp_path):
    ref = C.load_model(FIX / "ivf_small.dpq")
    ids = np.asarray(ref.sorted_ids_).copy()
    ids[3] = ids[4]  # a duplicate: not a permutation
    bad = IVFIndex.from_arrays(ref.quantizer.codebooks_, ref.quantizer.derived_codebooks_, ref.centers_,
                               ref.offsets_, np.asarray(ref.sorted_codes_), ids, cell_of=np.asarray(ref.cell_of_))
    bad.quantizer = ref.quantizer
    p = tmp_path / "perm.dpq"
    C.save_model(bad, p)
    with pytest.raises(InvariantError, match="do not partition"):
        C.load_model(p)
    cells = np.asarray(ref.cell_of_).copy()
    j = int(np.flatnonzero(cells != cells[0])[0])
    cells[j] = cells[0]
    bad2 = IVFIndex.from_arrays(ref.quantizer.codebooks_, ref.quantizer.derived_codebooks_, ref.centers_,
                                ref.offsets_, np.asarray(ref.sorted_codes_), np.asarray(ref.sorted_ids_),
                                cell_of=cells)
    bad2.quantizer = ref.quantizer
    p2 = tmp_path / "cells.dpq"
    C.save_model(bad2, p2)
    with pytest.raises(InvariantError, match="offsets disagree"):
        C.load_model(p2)


def test_baseline_shape_flat_round_trip(tmp_path):
    """PQ 4x16 / derived 4x8 over 2M codes (16 MB of codes, the configs[1]
    layout): save_model -> load_model (device CRC over every byte) ->
    identical search to the in-memory index."""
    from conftest import c1_codebooks, load_golden

    g = load_golden("c1_sampled")
    cb = c1_codebooks(g)
    rng = np.random.default_rng(7)
    codes = rng.integers(0, 65536, size=(2_000_000, 4), dtype=np.uint16)
    codes[: g["codes"].shape[0]] = g["codes"]
    mem = FlatIndex.from_arrays(cb, g["derived"], codes)
    mem.quantizer._kind = "pq"
    mem.quantizer._params = {"m": 4, "b": 16, "bbar": 8, "seed": 42, "max_iters": 50}
    mem.quantizer.distortions_ = np.zeros(4)
    p = tmp_path / "c2shape.dpq"
    C.save_model(mem, p)
    idx = C.load_model(p)
    st = C.load_model.last_stats
    assert st["bytes"] == codes.nbytes
    Y = g["queries"][:32]
    d0, i0 = mem.search(Y, 100, mode="derived", r2=1000)
    d1, i1 = idx.search(Y, 100, mode="derived", r2=1000)
    np.testing.assert_array_equal(i0, i1)
    np.testing.assert_array_equal(d0, d1)
