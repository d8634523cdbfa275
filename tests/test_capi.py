"""The C-ABI library loads and exports every symbol include/tftb200.h
declares (no compute calls: this runs without a GPU)."""

import os
import re

from paper_1001_5272_b200 import backend

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    with open(os.path.join(ROOT, "include", "tftb200.h")) as f:
        src = f.read()
    return set(re.findall(r"\b(tftb_\w+)\s*\(", src))


def test_header_symbols_exported():
    lib = backend.load()
    names = declared()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
    assert set(backend.SIGNATURES) == names


def test_version_and_counters():
    lib = backend.load()
    assert b"sm_100a" in lib.tftb_version()
    assert backend.launch_count(reset=True) >= 0
    backend.aux_bytes(reset=True)
    assert backend.aux_bytes() == 0  # nothing allocated without a call
