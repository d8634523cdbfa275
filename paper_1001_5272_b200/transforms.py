"""In-place forward / inverse truncated Fourier transforms on the B200.

Same public surface, argument checks and output order as the reference
(pkg/src/tftmul/transforms.py:208-256): tft(buf, cfg) overwrites buf[s]
with F(omega_s) for s < n, itft undoes it exactly, fft_pow2 is tft
restricted to powers of two.  Validation happens here, before dispatch, in
the reference's order (transforms.py:28-34): ValueError for an empty buffer,
UnsupportedSizeError for n > 2^K.

Every call runs on the GPU through libtftb200 (backend.py); there is no
CPU fallback.  Buffers the kernels cannot view in place (lists, tuples,
array('I'), ...) are staged through an array('Q') copy and written back, so
the result is still the GPU's.  The reference's `trace` argument forces its
pure-Python walk (transforms.py:218, 231); a level-synchronous GPU
schedule has no node walk to trace, so a trace request raises.
"""

from array import array

from . import backend
from .modring import UnsupportedSizeError


# Longest transform the device plans cover: two passes over 2^14-word tiles
# reach 2^28 words (host.h make_plan), and n = 2^28 + r, r <= 4, runs as the
# 2^28 transform plus r dot products (p2r.cuh).  Rings with K > 28
# (3221225473: K = 30; the 62-bit prime: K = 57) accept longer lengths in
# the reference; here they raise UnsupportedSizeError, the reference's own
# exception for lengths a config cannot transform (transforms.py:28-34).
DEVICE_MAX_LOG = 28
DEVICE_P2R_MAX = 4


def device_supports(n):
    return n <= (1 << DEVICE_MAX_LOG) or n - (1 << DEVICE_MAX_LOG) <= DEVICE_P2R_MAX


def _check_size(n, cfg):
    if n == 0:
        raise ValueError("cannot transform an empty buffer")
    if n > 1 << cfg.K:
        raise UnsupportedSizeError(f"length {n} exceeds the 2^{cfg.K} roots the config supports")
    if not device_supports(n):
        raise UnsupportedSizeError(f"length {n} exceeds the B200 plans' 2^{DEVICE_MAX_LOG}(+{DEVICE_P2R_MAX}) words")


def _credit(cfg, mults, adds):
    c = cfg.counters
    if c is not None:
        c.mults += mults
        c.adds += adds


def _no_trace(trace):
    if trace is not None:
        raise NotImplementedError("node traces come from the reference's CPU walk; "
                                  "the B200 path runs a level-synchronous schedule")


def _run(buf, cfg, call):
    n = len(buf)
    mv = backend.kernel_view(buf)
    if mv is not None:
        m, a = call(mv, n)
    else:
        staged = array("Q", buf)
        m, a = call(memoryview(staged), n)
        for i, v in enumerate(staged):
            buf[i] = v
    _credit(cfg, m, a)


def tft(buf, cfg, trace=None):
    """In-place forward transform of an arbitrary-length buffer."""
    _no_trace(trace)
    _check_size(len(buf), cfg)
    K = backend.kernels()
    _run(buf, cfg, lambda mv, n: K.tft(mv, 0, n, cfg.p, cfg.omegaK, cfg.K))


def itft(buf, cfg, trace=None):
    """In-place inverse transform; exact inverse of tft on the same config."""
    _no_trace(trace)
    _check_size(len(buf), cfg)
    K = backend.kernels()
    _run(buf, cfg, lambda mv, n: K.itft(mv, 0, n, cfg.p, cfg.omegaK, cfg.K, cfg.inv2))


def fft_pow2(buf, cfg):
    """Forward transform restricted to power-of-two lengths."""
    n = len(buf)
    _check_size(n, cfg)
    if n & (n - 1):
        raise ValueError(f"length {n} is not a power of two")
    K = backend.kernels()
    _run(buf, cfg, lambda mv, n: K.tft(mv, 0, n, cfg.p, cfg.omegaK, cfg.K))
