"""CPU checks of the C-ABI boundary: the library loads and exports every
symbol include/tneat.h declares (no compute -- there is no GPU here)."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "tneat.h")


def declared_symbols() -> list[str]:
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(an_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared_symbols()
    assert "an_transform" in names and "an_forward" in names
    assert len(names) >= 4


def test_library_exports_every_declared_symbol():
    from paper_2404_01817_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libtneat.so not built")
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, f"symbols declared in tneat.h but not exported: {missing}"
    # the ctypes signature table covers exactly the declared ABI
    assert sorted(_native.SIGNATURES) == declared_symbols()


def test_program_stride_is_host_callable():
    from paper_2404_01817_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libtneat.so not built")
    s32 = _native.lib().an_program_stride(128, 512, 8, 0)
    s64 = _native.lib().an_program_stride(128, 512, 8, 1)
    assert s32 % 16 == 0 and s64 > s32
    # header 32 + out slots 16 + groups 16N + steps 16N + u16 src / f32 w x (3C+12N+16)
    e = 3 * 512 + 12 * 128 + 16
    assert s32 == 32 + 16 + 128 * 16 + 128 * 16 + 2 * e + 4 * e
