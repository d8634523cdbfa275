"""The drop-in native boundary: libtftb200.so (sm_100a) through ctypes.

Mirrors reference pkg/src/tftmul/backend.py:27-54: `kernels()` returns the
module-like object the transforms call, `backend_name()` names it, and
`kernel_view()` screens caller buffers exactly as the reference does (1-D,
8-byte items, C-contiguous, writable unless told otherwise, format Q/L/N).
The object returned by kernels() has the reference `_kernels` signatures
(_kernels.pyx:415-480):

    tft(x, off, n, p, top, K) -> (mults, adds)
    itft(x, off, n, p, top, K, inv2) -> (mults, adds)
    multiply(a, b, x, p, top, K, inv2) -> (mults, adds)

but runs on the GPU.  There is no CPU fallback: if the shared library is
missing, or the CUDA call fails, these raise.  ctypes releases the GIL for
the duration of each call, like the reference's `with nogil` blocks.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TFTB_LIB: an alternative build of the same library (tools/build_variant.py experiments)
LIB_PATH = os.environ.get("TFTB_LIB") or os.path.join(_HERE, "libtftb200.so")

_forced = os.environ.get("TFTMUL_BACKEND", "").strip().lower()
if _forced in ("py", "pure", "python"):
    raise ImportError("this build has no CPU path; TFTMUL_BACKEND=pure is not available")
if _forced not in ("", "auto", "c", "ext", "compiled", "b200", "cuda"):
    raise ImportError(f"unknown TFTMUL_BACKEND value {_forced!r}")

_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p

# every symbol include/tftb200.h declares, with its ctypes signature
SIGNATURES = {
    "tftb_tft_u64": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                    _i64p, _i64p]),
    "tftb_itft_u64": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                     ctypes.c_uint64, _i64p, _i64p]),
    "tftb_multiply_u64": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, ctypes.c_int64, _vp, ctypes.c_uint64,
                                         ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, _i64p, _i64p]),
    "tftb_tft_batch_u64": (ctypes.c_int, [_vp, _i64p, _i64p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_int, ctypes.c_int]),
    "tftb_horner_u64": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, _u64p]),
    "tftb_fold_twist_u64": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_uint64,
                                           ctypes.c_uint64]),
    "tftb_ring_get": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(_vp)]),
    "tftb_ring_word_bytes": (ctypes.c_int, [_vp]),
    "tftb_tft_dev": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _i64p, _i64p,
                                    ctypes.c_int, _vp]),
    "tftb_plan_create": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _i64p, _i64p,
                                        ctypes.POINTER(_vp)]),
    "tftb_plan_execute": (ctypes.c_int, [_vp, _vp, ctypes.c_int, _vp]),
    "tftb_plan_destroy": (ctypes.c_int, [_vp]),
    "tftb_multiply_dev": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_int64, _vp, ctypes.c_int64,
                                         ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int64, _vp, _vp]),
    "tftb_words_from_u64": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, _vp]),
    "tftb_words_to_u64": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, _vp]),
    "tftb_last_error": (ctypes.c_char_p, []),
    "tftb_version": (ctypes.c_char_p, []),
    "tftb_launch_count": (ctypes.c_int64, [ctypes.c_int]),
    "tftb_aux_bytes": (ctypes.c_int64, [ctypes.c_int]),
    "tftb_stage_bytes": (ctypes.c_int64, [ctypes.c_int]),
    "tftb_tally_transform": (ctypes.c_int, [ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, _i64p, _i64p]),
    "tftb_tally_multiply": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, _i64p,
                                           _i64p]),
}

_lib = None


class NativeError(RuntimeError):
    """A CUDA or argument failure reported by libtftb200."""


def load():
    """Load libtftb200.so (raises ImportError if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc):
    if rc != 0:
        raise NativeError(load().tftb_last_error().decode())


def _addr(mv):
    """Address of a 1-D 8-byte buffer (read-only buffers allowed)."""
    if len(mv) == 0:
        return None
    return np.frombuffer(mv, dtype=np.uint64).ctypes.data


class _Kernels:
    """Module-like façade with the reference `_kernels` call signatures."""

    @staticmethod
    def tft(x, off, n, p, top, K):
        m, a = ctypes.c_int64(0), ctypes.c_int64(0)
        base = _addr(x) + 8 * off
        check(load().tftb_tft_u64(base, n, p, top, K, ctypes.byref(m), ctypes.byref(a)))
        return m.value, a.value

    @staticmethod
    def itft(x, off, n, p, top, K, inv2):
        m, a = ctypes.c_int64(0), ctypes.c_int64(0)
        base = _addr(x) + 8 * off
        check(load().tftb_itft_u64(base, n, p, top, K, inv2, ctypes.byref(m), ctypes.byref(a)))
        return m.value, a.value

    @staticmethod
    def multiply(a, b, x, p, top, K, inv2):
        m, ad = ctypes.c_int64(0), ctypes.c_int64(0)
        check(load().tftb_multiply_u64(_addr(a), len(a), _addr(b), len(b), _addr(x), p, top, K, inv2,
                                       ctypes.byref(m), ctypes.byref(ad)))
        return m.value, ad.value


_KERNELS = _Kernels()


def kernels():
    load()
    return _KERNELS


def backend_name():
    return "b200"


def kernel_view(buf, writable=True):
    """A memoryview the kernels accept, or None (reference backend.py:35-54)."""
    try:
        mv = memoryview(buf)
    except TypeError:
        return None
    if mv.ndim != 1 or mv.itemsize != 8 or not mv.contiguous:
        return None
    if writable and mv.readonly:
        return None
    if mv.format not in ("Q", "L", "N", "<Q", "=Q", "<L", "=L"):
        return None
    if mv.format != "Q":
        try:
            mv = mv.cast("B").cast("Q")
        except TypeError:
            return None
    return mv


def ring_handle(cfg):
    """Opaque device ring (twiddle tables) for a RingConfig, cached natively."""
    h = _vp()
    check(load().tftb_ring_get(cfg.p, cfg.omegaK, cfg.K, ctypes.byref(h)))
    return h


def launch_count(reset=False):
    return int(load().tftb_launch_count(1 if reset else 0))


def stage_bytes(reset=False):
    """Device bytes this thread's host-pointer calls allocated for the
    caller's words (high-water mark since the last reset)."""
    return int(load().tftb_stage_bytes(1 if reset else 0))


def aux_bytes(reset=False):
    """Device bytes this thread's calls allocated beyond the transformed
    words (high-water mark since the last reset): the footprint audit."""
    return int(load().tftb_aux_bytes(1 if reset else 0))
