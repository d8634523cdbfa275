"""Op tallies: the (mults, adds) the reference kernels return for a call
(`_kernels.pyx:415-480`), reproduced by the host-side model in
csrc/tally.h, against tests/golden/tallies.json (written by the reference's
compiled kernels, tests/golden/make_golden.py --tallies).  Host-only entry
points: no GPU needed."""

import ctypes
import json
import os

import pytest

from paper_1001_5272_b200 import backend

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def tallies():
    with open(os.path.join(HERE, "golden", "tallies.json")) as f:
        return json.load(f)


def _tally(n, p, K, inverse):
    m, a = ctypes.c_int64(), ctypes.c_int64()
    backend.check(backend.load().tftb_tally_transform(n, p, K, inverse, ctypes.byref(m), ctypes.byref(a)))
    return [m.value, a.value]


def _tally_mul(la, lb, p, K):
    m, a = ctypes.c_int64(), ctypes.c_int64()
    backend.check(backend.load().tftb_tally_multiply(la, lb, p, K, ctypes.byref(m), ctypes.byref(a)))
    return [m.value, a.value]


def test_transform_tallies_match_reference(golden, tallies):
    assert len(tallies["transforms"]) > 340
    for case in tallies["transforms"]:
        p, _, K = golden["primes"][case["prime"]]
        assert _tally(case["n"], p, K, 0) == case["tft"], case
        assert _tally(case["n"], p, K, 1) == case["itft"], case


def test_product_tallies_match_reference(golden, tallies):
    for case in tallies["products"]:
        p, _, K = golden["primes"][case["prime"]]
        assert _tally_mul(case["la"], case["lb"], p, K) == case["tally"], case


def test_tally_rejects_empty():
    with pytest.raises(backend.NativeError):
        _tally(0, 998244353, 23, 0)
    with pytest.raises(backend.NativeError):
        _tally_mul(0, 5, 998244353, 23)
