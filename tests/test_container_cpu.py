"""Model containers, host side: the file format against
the reference's own containers (tests/golden/containers, written by
derivedpq.save_model), the mirror's save_model byte for byte, the
reference's FormatError / InvariantError cases, and a numpy restatement of
the device CRC-32 algorithm of dpq_container.cu checked against zlib (the
algebra the kernel relies on; the kernel itself is checked on the GPU in
test_gpu_container.py)."""

from __future__ import annotations

import json
import struct
import zlib
from pathlib import Path

import numpy as np
import pytest

from paper_1905_06900_b200 import FormatError, InvariantError
from paper_1905_06900_b200 import container as C
from paper_1905_06900_b200.flat import ArrayQuantizer, FlatIndex
from paper_1905_06900_b200.ivf import IVFIndex

FIX = Path(__file__).resolve().parent / "golden" / "containers"
CASES = ["pq_small", "flat_u8", "flat_u16", "flat_opq", "ivf_small"]


# ------------------------------------------------ device CRC, restated --

P = 0xEDB88320
_T = np.zeros(256, np.uint32)
for _i in range(256):
    _c = _i
    for _ in range(8):
        _c = (_c >> 1) ^ (P if _c & 1 else 0)
    _T[_i] = _c


def _apply(cols, v):
    v = np.asarray(v, np.uint32)
    r = np.zeros_like(v)
    for b in range(32):
        r ^= np.where((v >> np.uint32(b)) & np.uint32(1), cols[b], np.uint32(0)).astype(np.uint32)
    return r


def _mul(a, b):
    return _apply(a, b)


_A1 = np.array([((1 << b) >> 8) ^ int(_T[(1 << b) & 0xFF]) for b in range(32)], np.uint32)
_POW = [_A1]
for _ in range(31):
    _POW.append(_mul(_POW[-1], _POW[-1]))
ORDER = 0xFFFFFFFF


def _adv_mat(n):
    r = np.array([1 << b for b in range(32)], np.uint32)
    n %= ORDER
    i = 0
    while n:
        if n & 1:
            r = _mul(_POW[i], r)
        n >>= 1
        i += 1
    return r


def _adv(v, n):
    return _apply(_adv_mat(n), v)


def _sliced_tab(mat):
    return np.stack([_apply(mat, np.arange(256, dtype=np.uint32) << np.uint32(8 * k)) for k in range(4)])


def _sliced(t, v):
    return t[0][v & 255] ^ t[1][(v >> 8) & 255] ^ t[2][(v >> 16) & 255] ^ t[3][v >> 24]


THREADS, GROUPS = 256, 64
STRIDE = THREADS * 16
CHUNK = STRIDE * GROUPS
T4, TJ = _sliced_tab(_adv_mat(4)), _sliced_tab(_adv_mat(STRIDE - 12))
TREE = [_adv_mat(16 << k) for k in range(5)]
W512 = _adv_mat(512)


def chunk_raw(chunk: bytes) -> int:
    """One CTA of k_crc_chunks: thread t absorbs the words at 16 t + 4096 g,
    shuffle tree over lanes, A_512 chain over warps -> raw CRC at the chunk end."""
    w = np.frombuffer(chunk, "<u4").reshape(GROUPS, THREADS, 4)
    s = np.zeros(THREADS, np.uint32)
    for g in range(GROUPS):
        for k in range(4):
            t = TJ if (k == 3 and g < GROUPS - 1) else T4
            s = _sliced(t, s ^ w[g, :, k])
    s = s.reshape(8, 32).copy()
    lane = np.arange(32)
    for k in range(5):
        mask = (2 << k) - 1
        o = np.concatenate([s[:, :1 << k], s[:, :32 - (1 << k)]], axis=1)  # __shfl_up_sync
        moved = _apply(TREE[k], o.reshape(-1)).reshape(8, 32)
        s = np.where((lane & mask) == mask, s ^ moved, s)
    v = s[0, 31]
    for wv in s[1:, 31]:
        v = _apply(W512, v) ^ wv
    return int(v)


def device_crc_model(data: bytes) -> int:
    full = len(data) // CHUNK
    tail = len(data) - full * CHUNK
    acc0 = 0
    for c in range(full):
        acc0 ^= int(_adv(chunk_raw(data[c * CHUNK:(c + 1) * CHUNK]), (full - 1 - c) * CHUNK + tail))
    acc1 = chunk_raw(data[full * CHUNK:] + bytes(CHUNK - tail)) if tail else 0
    z = CHUNK - tail if tail else 0
    raw = acc0 ^ int(_adv(acc1, ORDER - (z % ORDER)))
    return (~(int(_adv(0xFFFFFFFF, len(data))) ^ raw)) & 0xFFFFFFFF


@pytest.mark.parametrize("n", [0, 1, 3, 16, 4095, CHUNK, CHUNK + 5, 2 * CHUNK + 4100])
def test_device_crc_algorithm_equals_zlib(n):
    data = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8).tobytes()
    assert device_crc_model(data) == zlib.crc32(data)


def test_crc_order_of_x_is_2_32_minus_1():
    assert np.array_equal(_adv_mat(ORDER), np.array([1 << b for b in range(32)], np.uint32))


# --------------------------------------------------------- file format --

@pytest.mark.parametrize("case", CASES)
def test_reference_container_layout(case):
    path = FIX / f"{case}.dpq"
    kind, params, manifest, start, size = C.read_header(path)
    arrs = C.layout(manifest, start)
    assert arrs[-1][3] + arrs[-1][4] == size  # arrays tile the file exactly
    _, _, arrays = C.read_arrays(path)
    for name, _, _, _, _, crc in arrs:
        assert zlib.crc32(np.ascontiguousarray(arrays[name]).tobytes()) == crc
    assert kind == {"pq_small": "pq", "flat_opq": "flat", "ivf_small": "ivf"}.get(case, "flat")


def _mirror_from_arrays(kind, params, arrays):
    """Mirror objects (host arrays) the way load_model assembles them."""
    if kind in ("pq", "opq"):
        return C._quantizer(kind, params, arrays)
    q = C._quantizer(params["quantizer_kind"], params["quantizer_params"],
                     {k[2:]: v for k, v in arrays.items() if k.startswith("q.")})
    if kind == "flat":
        idx = FlatIndex(q)
        idx.codes_ = arrays["codes"]
        idx.n_ = idx.codes_.shape[0]
        return idx
    idx = IVFIndex(q, n_cells=params["n_cells"], seed=params["seed"], coarse_iters=params["coarse_iters"])
    for k in ("centers", "cell_of", "sorted_ids", "sorted_codes", "offsets"):
        setattr(idx, k + "_", arrays[k])
    idx.n_ = idx.sorted_ids_.shape[0]
    return idx


@pytest.mark.parametrize("case", CASES)
def test_save_model_writes_the_reference_bytes(case, tmp_path):
    path = FIX / f"{case}.dpq"
    model = _mirror_from_arrays(*C.read_arrays(path))
    out = tmp_path / "again.dpq"
    C.save_model(model, out)
    assert out.read_bytes() == path.read_bytes()


def test_quantizer_container_loads_on_host(tmp_path):
    q = C.load_model(FIX / "pq_small.dpq")
    _, _, arrays = C.read_arrays(FIX / "pq_small.dpq")
    assert isinstance(q, ArrayQuantizer)
    np.testing.assert_array_equal(q.codebooks_, arrays["codebooks"])
    np.testing.assert_array_equal(q.derived_codebooks_, arrays["derived_codebooks"])
    assert q.code_dtype_ == np.uint8 and q.b == 4


# --------------------------------------------- the reference's errors --

def test_wrong_magic(tmp_path):
    p = tmp_path / "bad.dpq"
    p.write_bytes(b"NOPE" + b"\x00" * 32)
    with pytest.raises(FormatError, match="magic"):
        C.load_model(p)


def test_unsupported_version(tmp_path):
    blob = bytearray((FIX / "pq_small.dpq").read_bytes())
    blob[4:6] = struct.pack("<H", 2)
    p = tmp_path / "v2.dpq"
    p.write_bytes(bytes(blob))
    with pytest.raises(FormatError, match="unsupported container version 2"):
        C.load_model(p)


def test_corrupt_header(tmp_path):
    blob = bytearray((FIX / "pq_small.dpq").read_bytes())
    blob[10] = ord("!")
    p = tmp_path / "hdr.dpq"
    p.write_bytes(bytes(blob))
    with pytest.raises(FormatError, match="corrupt header"):
        C.load_model(p)


@pytest.mark.parametrize("case", ["pq_small", "flat_u8", "ivf_small"])
def test_truncated_container(case, tmp_path):
    p = tmp_path / "t.dpq"
    p.write_bytes((FIX / f"{case}.dpq").read_bytes()[:-10])
    kind, _, manifest, start, _ = C.read_header(p)
    last = manifest[-1]["name"]
    with pytest.raises(FormatError, match=f"truncated array '{last}'"):
        C.load_model(p)


def test_checksum_catches_flipped_array_byte(tmp_path):
    blob = bytearray((FIX / "pq_small.dpq").read_bytes())
    blob[-40] ^= 0xFF
    p = tmp_path / "flip.dpq"
    p.write_bytes(bytes(blob))
    with pytest.raises(FormatError, match="checksum"):
        C.load_model(p)
    assert C.load_model(p, verify=False) is not None


def test_load_time_validation_catches_corruption(tmp_path):
    kind, params, arrays = C.read_arrays(FIX / "pq_small.dpq")
    arrays = {k: v.copy() for k, v in arrays.items()}
    arrays["derived_assignments"][0, 0] ^= 1
    p = tmp_path / "corrupt.dpq"
    C.save_model(C._quantizer(kind, params, arrays), p)
    with pytest.raises(InvariantError):
        C.load_model(p)
    assert C.load_model(p, verify=False) is not None


def test_unknown_kind(tmp_path):
    blob = (FIX / "pq_small.dpq").read_bytes()
    hlen = struct.unpack("<I", blob[6:10])[0]
    header = json.loads(blob[10:10 + hlen])
    header["kind"] = "lsh"
    h = json.dumps(header).encode()
    p = tmp_path / "kind.dpq"
    p.write_bytes(blob[:4] + struct.pack("<HI", 1, len(h)) + h + blob[10 + hlen:])
    with pytest.raises(FormatError, match="unknown model kind 'lsh'"):
        C.load_model(p)
