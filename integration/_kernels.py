"""tftmul/_kernels.py -- drop-in replacement for the reference's Cython
extension (`_kernels.pyx:415-480`) that runs every call on the B200 through
libtftb200.so (include/tftb200.h).  Copy this file into the reference
package as `tftmul/_kernels.py`; the reference's
`backend.py:10-13` imports it, `backend_name()` reports "compiled", and
transforms.tft / itft / fft_pow2 and polymul.multiply call it unchanged.

The library is found through $TFTB_LIB, else next to this repository's
package (paper_1001_5272_b200/libtftb200.so).  ctypes releases the GIL for
each call, like the reference's `with nogil` blocks.
"""

import ctypes
import os

import numpy as np

_path = os.environ.get("TFTB_LIB") or os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1001_5272_b200", "libtftb200.so")
_lib = ctypes.CDLL(_path)
_i64p = ctypes.POINTER(ctypes.c_int64)
_vp, _u64, _i64, _int = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int
_lib.tftb_tft_u64.argtypes = [_vp, _i64, _u64, _u64, _int, _i64p, _i64p]
_lib.tftb_itft_u64.argtypes = [_vp, _i64, _u64, _u64, _int, _u64, _i64p, _i64p]
_lib.tftb_multiply_u64.argtypes = [_vp, _i64, _vp, _i64, _vp, _u64, _u64, _int, _u64, _i64p, _i64p]
_lib.tftb_last_error.restype = ctypes.c_char_p


def _addr(mv):
    return np.frombuffer(mv, dtype=np.uint64).ctypes.data if len(mv) else None


def _ok(rc):
    if rc:
        raise RuntimeError(_lib.tftb_last_error().decode())


def tft(x, off, n, p, top, K):                        # _kernels.pyx:415-421
    m, a = ctypes.c_int64(), ctypes.c_int64()
    _ok(_lib.tftb_tft_u64(_addr(x) + 8 * off, n, p, top, K, ctypes.byref(m), ctypes.byref(a)))
    return m.value, a.value


def itft(x, off, n, p, top, K, inv2):                 # _kernels.pyx:424-430
    m, a = ctypes.c_int64(), ctypes.c_int64()
    _ok(_lib.tftb_itft_u64(_addr(x) + 8 * off, n, p, top, K, inv2, ctypes.byref(m), ctypes.byref(a)))
    return m.value, a.value


def multiply(a, b, x, p, top, K, inv2):               # _kernels.pyx:433-480
    m, ad = ctypes.c_int64(), ctypes.c_int64()
    _ok(_lib.tftb_multiply_u64(_addr(a), len(a), _addr(b), len(b), _addr(x), p, top, K, inv2,
                               ctypes.byref(m), ctypes.byref(ad)))
    return m.value, ad.value
