"""Device-resident, batched entry points (torch tensors as device buffers).

The host-buffer API in transforms/polymul mirrors the reference one call at a
time; these wrappers expose the batched C ABI (include/tftb200.h
tftb_tft_dev / tftb_multiply_dev) so a whole batch of vectors or products
runs with the data already resident in HBM.  torch is only the allocator and
stream provider; the work is libtftb200's.

Device words: uint32 bit patterns in an int32 tensor when p < 2^32,
int64 (uint64 bit patterns) otherwise.
"""

import ctypes

import numpy as np
import torch

from . import backend
from .modring import UnsupportedSizeError
from .transforms import DEVICE_MAX_LOG, device_supports


def word_dtype(cfg):
    return torch.int32 if cfg.p < (1 << 32) else torch.int64


def word_np(cfg):
    return np.uint32 if cfg.p < (1 << 32) else np.uint64


def to_words(values, cfg, device="cuda"):
    """numpy/array('Q') residues -> device word tensor."""
    a = np.ascontiguousarray(np.asarray(values, dtype=np.uint64).astype(word_np(cfg)))
    t = torch.from_numpy(a.view(np.int32 if a.dtype == np.uint32 else np.int64))
    return t.to(device)


def from_words(t, cfg):
    """device word tensor -> numpy uint64 residues."""
    a = t.detach().cpu().numpy()
    return a.view(np.uint32 if a.dtype == np.int32 else np.uint64).astype(np.uint64)


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _check_words(t, cfg):
    if not isinstance(t, torch.Tensor) or not t.is_cuda or not t.is_contiguous() or t.dtype != word_dtype(cfg):
        raise ValueError(f"expected a contiguous CUDA {word_dtype(cfg)} tensor")


def _check_lengths(ln, cfg):
    if (ln <= 0).any() or (ln > (1 << cfg.K)).any():
        raise ValueError("vector lengths must lie in [1, 2^K]")
    big = ln[ln > (1 << DEVICE_MAX_LOG)]
    if big.size and not all(device_supports(int(n)) for n in big):
        raise UnsupportedSizeError(f"vector lengths beyond the B200 plans' 2^{DEVICE_MAX_LOG} words")


def _ragged_layout(lengths, offsets):
    """Validated (lengths, offsets) int64 arrays: offsets >= 0 and no two
    vectors overlapping (include/tftb200.h: vectors must not overlap)."""
    ln = np.ascontiguousarray(lengths, dtype=np.int64).ravel()
    if offsets is None:
        of = np.concatenate(([0], np.cumsum(ln)[:-1])).astype(np.int64) if ln.size else ln.copy()
    else:
        of = np.ascontiguousarray(offsets, dtype=np.int64).ravel()
        if of.size != ln.size:
            raise ValueError("offsets and lengths differ in size")
        if (of < 0).any():
            raise ValueError("negative vector offset")
        order = np.argsort(of, kind="stable")
        so, sl = of[order], ln[order]
        if so.size > 1 and (so[1:] < so[:-1] + sl[:-1]).any():
            raise ValueError("vectors overlap")
    return ln, of


def tft_batch_(data, cfg, n=None, count=1, stride=None, lengths=None, offsets=None, inverse=False,
               stream=None):
    """In-place (I)TFT of `count` vectors inside `data`.

    Either uniform (n, count, stride = n by default) or ragged (lengths and
    offsets: host int64 sequences).  Asynchronous on `stream`."""
    _check_words(data, cfg)
    h = backend.ring_handle(cfg)
    lib = backend.load()
    if lengths is not None:
        ln, of = _ragged_layout(lengths, offsets)
        count = ln.size
        _check_lengths(ln, cfg)
        if count and int((of + ln).max()) > data.numel():
            raise ValueError("vectors run past the end of the buffer")
        backend.check(lib.tftb_tft_dev(h, ctypes.c_void_p(data.data_ptr()), count, 0, 0,
                                       of.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                       ln.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                       1 if inverse else 0, _stream(stream)))
        return data
    if n is None or n <= 0 or n > (1 << cfg.K):
        raise ValueError("n must lie in [1, 2^K]")
    _check_lengths(np.array([n]), cfg)
    if count < 0:
        raise ValueError("negative vector count")
    stride = n if stride is None else stride
    if count > 1 and stride < n:
        raise ValueError("stride shorter than the vector length (vectors overlap)")
    if count and (count - 1) * stride + n > data.numel():
        raise ValueError("vectors run past the end of the buffer")
    backend.check(lib.tftb_tft_dev(h, ctypes.c_void_p(data.data_ptr()), count, n, stride, None, None,
                                   1 if inverse else 0, _stream(stream)))
    return data


def multiply_batch(a, b, x, cfg, count, la, lb, scratch=None, stream=None):
    """x[v] <- a[v] * b[v] for `count` pairs stored back to back
    (a: count*la words, b: count*lb, x: count*(la+lb-1))."""
    for t in (a, b, x):
        _check_words(t, cfg)
    if count < 0 or la <= 0 or lb <= 0:
        raise ValueError("need count >= 0 and non-empty operands")
    r = la + lb - 1
    if r > (1 << cfg.K):
        raise UnsupportedSizeError("product length exceeds 2^K")
    if not device_supports(r):
        raise UnsupportedSizeError(f"product length beyond the B200 plans' 2^{DEVICE_MAX_LOG} words")
    if a.numel() < count * la or b.numel() < count * lb or x.numel() < count * r:
        raise ValueError("buffers too small for the batch")
    if scratch is not None:
        _check_words(scratch, cfg)
        if scratch.numel() < count * r:
            raise ValueError(f"scratch needs count*(la+lb-1) = {count * r} words")
    sp = ctypes.c_void_p(scratch.data_ptr()) if scratch is not None else None
    h = backend.ring_handle(cfg)
    backend.check(backend.load().tftb_multiply_dev(h, ctypes.c_void_p(a.data_ptr()), la, la,
                                                   ctypes.c_void_p(b.data_ptr()), lb, lb,
                                                   ctypes.c_void_p(x.data_ptr()), r, count, sp,
                                                   _stream(stream)))
    return x


class BatchPlan:
    """A reusable grouping of a ragged batch (tftb_plan_*): build once, then
    execute() issues only kernel launches on the given stream."""

    def __init__(self, cfg, lengths, offsets=None):
        ln, of = _ragged_layout(lengths, offsets)
        if ln.size == 0:
            raise ValueError("a plan needs at least one vector")
        _check_lengths(ln, cfg)
        self.cfg = cfg
        self.count = int(ln.size)
        self.span = int((of + ln).max()) if ln.size else 0
        self._lib = backend.load()
        self._h = ctypes.c_void_p()
        backend.check(self._lib.tftb_plan_create(backend.ring_handle(cfg), self.count, 0, 0,
                                                 of.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                                 ln.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                                 ctypes.byref(self._h)))

    def execute(self, data, inverse=False, stream=None):
        _check_words(data, self.cfg)
        if data.numel() < self.span:
            raise ValueError("buffer smaller than the plan's vectors")
        backend.check(self._lib.tftb_plan_execute(self._h, ctypes.c_void_p(data.data_ptr()),
                                                  1 if inverse else 0, _stream(stream)))
        return data

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.tftb_plan_destroy(h)
            self._h = None
