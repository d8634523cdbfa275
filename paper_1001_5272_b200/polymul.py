"""Polynomial product over Z/pZ on the B200.

Same public surface and validation order as the reference's Algorithm-3
entry point (pkg/src/tftmul/polymul.py:111-141): multiply(A, B, X, cfg)
writes the len(A)+len(B)-1 product coefficients into X, never writes A or
B, and raises ValueError for empty inputs, a wrong output length or an
aliased output, and UnsupportedSizeError when the product is longer than 2^K.

The device computes X^ = TFT_r(A), Y^ = TFT_r(B) (r = len(X)), the
pointwise product and one in-place ITFT_r -- the three-transform
formulation BASELINE config 4 describes.  Because the arithmetic is exact
the coefficients are identical to the reference's Algorithm 3 (its
pre-inverse state is the same DFT, reference tests/test_polymul.py:143-168).
block_schedule is the reference's greedy power-of-two cover (polymul.py:25-36),
kept for API parity; the device does not need it.  horner_eval and
fold_twist, the reference's Algorithm-3 helpers (polymul.py:39-88), run on
the device too (csrc/poly.cu), so the module's whole public surface is GPU.
"""

from array import array
from typing import NamedTuple

from . import backend
from .modring import UnsupportedSizeError
from .modring import omega
from .transforms import DEVICE_MAX_LOG, _credit, device_supports


class BlockStep(NamedTuple):
    q: int
    ell: int
    L: int


def block_schedule(r):
    """Greedy cover of [0, r-1) by blocks L = 2^ell with L | q, 2L <= r-q < 4L."""
    q = 0
    while q < r - 1:
        ell = (r - q).bit_length() - 2
        yield BlockStep(q, ell, 1 << ell)
        q += 1 << ell


def _words(buf):
    """(address, keepalive) of a buffer's uint64 words, staged when the
    kernels cannot view it in place."""
    import numpy as np
    mv = backend.kernel_view(buf, writable=False)
    if mv is None:
        mv = memoryview(array("Q", buf))
    return (np.frombuffer(mv, dtype=np.uint64).ctypes.data if len(mv) else None), mv


def horner_eval(poly, point, cfg):
    """Evaluate a nonempty coefficient sequence at one ring point (reference
    polymul.py:39-52), on the GPU."""
    import ctypes
    if len(poly) == 0:
        raise ValueError("cannot evaluate an empty polynomial")
    addr, keep = _words(poly)
    out = ctypes.c_uint64(0)
    backend.check(backend.load().tftb_horner_u64(addr, len(keep), point % cfg.p, cfg.p, ctypes.byref(out)))
    n = len(poly) - 1
    _credit(cfg, n, n)
    return int(out.value)


def fold_twist(src, X, base, L, q, cfg):
    """Accumulate the twisted fold of src into the block X[base : base+L]
    (reference polymul.py:55-88): block slot i gains the sum of
    src[i + j*L] * omega(q)^(i + j*L) over j, on the GPU."""
    if L <= 0 or base < 0 or base + L > len(X):
        raise IndexError("fold block outside the output buffer")
    s_addr, s_keep = _words(src)
    w = omega(q, cfg) if q else 1
    mvx = backend.kernel_view(X)
    staged = None
    if mvx is None:
        staged = array("Q", X[base:base + L])
        mvx, off = memoryview(staged), 0
    else:
        off = base
    import numpy as np
    x_addr = np.frombuffer(mvx, dtype=np.uint64).ctypes.data + 8 * off
    backend.check(backend.load().tftb_fold_twist_u64(s_addr, len(s_keep), x_addr, L, w, cfg.p))
    if staged is not None:
        for i, v in enumerate(staged):
            X[base + i] = v
    ls = len(src)
    _credit(cfg, 2 * (ls - 1) if q and ls else 0, ls)


def multiply(A, B, X, cfg):
    """X <- A * B (coefficients), computed on the GPU."""
    la, lb = len(A), len(B)
    if la == 0 or lb == 0:
        raise ValueError("cannot multiply an empty polynomial")
    r = la + lb - 1
    if len(X) != r:
        raise ValueError(f"output buffer has length {len(X)}, need {r}")
    if r > 1 << cfg.K:
        raise UnsupportedSizeError(f"product length {r} exceeds the 2^{cfg.K} roots the config supports")
    if not device_supports(r):
        raise UnsupportedSizeError(f"product length {r} exceeds the B200 plans' 2^{DEVICE_MAX_LOG} words")
    if X is A or X is B:
        raise ValueError("output buffer must be distinct from the inputs")
    K = backend.kernels()
    mva = backend.kernel_view(A, writable=False)
    mvb = backend.kernel_view(B, writable=False)
    mvx = backend.kernel_view(X)
    ax = mva if mva is not None else memoryview(array("Q", A))
    bx = mvb if mvb is not None else memoryview(array("Q", B))
    staged = None
    if mvx is None:
        staged = array("Q", bytes(8 * r))
        mvx = memoryview(staged)
    m, a = K.multiply(ax, bx, mvx, cfg.p, cfg.omegaK, cfg.K, cfg.inv2)
    if staged is not None:
        for i, v in enumerate(staged):
            X[i] = v
    _credit(cfg, m, a)
