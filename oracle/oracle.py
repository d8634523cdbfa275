"""ORACLE — test infrastructure only (see oracle/__init__.py).

ctypes bindings for oracle/liboracle.so (the C restatement) and an importer
for oracle/_ref/_kernels (the reference's compiled Cython kernels,
`_kernels.pyx:415-480`).  Buffers are numpy uint64 arrays or array('Q').
"""

import ctypes
import glob
import importlib.util
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build():
    """Compile liboracle.so (and the reference kernels when the reference
    tree is present)."""
    subprocess.check_call(["make", "-s", "-C", _HERE, "all"])
    if os.path.exists("/root/reference/pkg/src/tftmul/_kernels.pyx"):
        subprocess.check_call(["make", "-s", "-C", _HERE, "ref"])


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        for name in ("orc_tft", "orc_itft"):
            f = getattr(L, name)
            f.argtypes = [_u64p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int]
            f.restype = ctypes.c_int
        L.orc_multiply.argtypes = [_u64p, ctypes.c_int64, _u64p, ctypes.c_int64, _u64p,
                                   ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int]
        L.orc_multiply.restype = ctypes.c_int
        L.orc_naive_dft.argtypes = [_u64p, ctypes.c_int64, _u64p, ctypes.c_uint64,
                                    ctypes.c_uint64, ctypes.c_int]
        L.orc_naive_dft.restype = ctypes.c_int
        L.orc_schoolbook.argtypes = [_u64p, ctypes.c_int64, _u64p, ctypes.c_int64, _u64p,
                                     ctypes.c_uint64]
        L.orc_schoolbook.restype = ctypes.c_int
        L.orc_omega.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int]
        L.orc_omega.restype = ctypes.c_uint64
        for name in ("orc_tft_batch", "orc_itft_batch"):
            f = getattr(L, name)
            f.argtypes = [_u64p, _i64p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64,
                          ctypes.c_int]
            f.restype = ctypes.c_int
        _LIB = L
    return _LIB


def _ptr(a):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(_u64p)


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"oracle {what} rejected its arguments")


def tft(x, p, top, K):
    """Forward TFT of a copy of x (numpy uint64), returns the new array."""
    y = np.ascontiguousarray(x, dtype=np.uint64).copy()
    _check(lib().orc_tft(_ptr(y), y.size, p, top, K), "tft")
    return y


def itft(x, p, top, K):
    y = np.ascontiguousarray(x, dtype=np.uint64).copy()
    _check(lib().orc_itft(_ptr(y), y.size, p, top, K), "itft")
    return y


def tft_batch(flat, lens, p, top, K, inverse=False):
    y = np.ascontiguousarray(flat, dtype=np.uint64).copy()
    ln = np.ascontiguousarray(lens, dtype=np.int64)
    f = lib().orc_itft_batch if inverse else lib().orc_tft_batch
    _check(f(_ptr(y), ln.ctypes.data_as(_i64p), ln.size, p, top, K), "batch")
    return y


def multiply(a, b, p, top, K):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    x = np.zeros(a.size + b.size - 1, dtype=np.uint64)
    _check(lib().orc_multiply(_ptr(a), a.size, _ptr(b), b.size, _ptr(x), p, top, K), "multiply")
    return x


def naive_dft(f, p, top, K):
    f = np.ascontiguousarray(f, dtype=np.uint64)
    out = np.zeros_like(f)
    _check(lib().orc_naive_dft(_ptr(f), f.size, _ptr(out), p, top, K), "naive_dft")
    return out


def schoolbook(a, b, p):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    out = np.zeros(a.size + b.size - 1, dtype=np.uint64)
    _check(lib().orc_schoolbook(_ptr(a), a.size, _ptr(b), b.size, _ptr(out), p), "schoolbook")
    return out


def omega(s, p, top, K):
    return int(lib().orc_omega(s, p, top, K))


def ref_kernels():
    """The reference's compiled kernels module (oracle/_ref), or None."""
    global _REF
    if _REF is None:
        hits = glob.glob(os.path.join(_HERE, "_ref", "_kernels*.so"))
        if not hits:
            return None
        spec = importlib.util.spec_from_file_location("_kernels", hits[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _REF = mod
    return _REF
