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


def _check_size(n, cfg):
    if n == 0:
        raise ValueError("cannot transform an empty buffer")
    if n > 1 << cfg.K:
        raise UnsupportedSizeError(f"length {n} exceeds the 2^{cfg.K} roots the config supports")


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
