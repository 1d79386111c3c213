"""The C-ABI library loads and exports every symbol include/dpq.h declares
(no compute calls: this runs without a GPU)."""

import re
from pathlib import Path

import pytest

from paper_1905_06900_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "dpq.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dpq_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared() == sorted(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for name in declared():
        assert hasattr(L, name), name


def test_abi_version_and_device_count():
    L = _lib.lib()
    assert L.dpq_abi_version() == 2
    assert _lib.device_count() >= 0


def test_no_device_fails_loudly():
    if _lib.device_count() > 0:
        pytest.skip("device present")
    with pytest.raises(RuntimeError, match="not available"):
        _lib.require_device(0)


def test_built_for_sm100a():
    so = Path(_lib.__file__).with_name("libdpq.so")
    data = so.read_bytes()
    assert b"sm_100a" in data or b"sm_100" in data
