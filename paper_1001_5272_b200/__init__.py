"""paper_1001_5272_b200 — B200-native in-place truncated Fourier transform.

Drop-in for the hot path of the reference package `tftmul` 0.1.0
(Harvey & Roche, arXiv 1001.5272): tft / itft / fft_pow2 / multiply with the
same RingConfig, root of unity, bit-reversed output order and exceptions
(reference pkg/src/tftmul/__init__.py).  The work runs in hand-written
sm_100a CUDA kernels (libtftb200.so, C ABI in include/tftb200.h); this
package is the host-side mirror of the reference interface.  Batched,
device-resident entry points live in `paper_1001_5272_b200.device`.
"""

from .backend import backend_name, kernel_view, kernels
from .modring import (
    OpCounters,
    RingConfig,
    RingConfigError,
    UnsupportedSizeError,
    ceil_lg,
    config_for_modulus,
    default_config,
    is_probable_prime,
    make_buffer,
    omega,
    revbin,
    revbin_increment,
    ring_add,
    ring_mul,
    ring_pow,
    ring_sub,
    root_of_level,
    zeros,
)
from .polymul import BlockStep, block_schedule, fold_twist, horner_eval, multiply
from .transforms import fft_pow2, itft, tft

__version__ = "0.1.0"

__all__ = [
    "BlockStep", "OpCounters", "RingConfig", "RingConfigError", "UnsupportedSizeError",
    "backend_name", "block_schedule", "ceil_lg", "config_for_modulus", "default_config",
    "fft_pow2", "fold_twist", "horner_eval", "is_probable_prime", "itft", "kernel_view", "kernels", "make_buffer",
    "multiply", "omega", "revbin", "revbin_increment", "ring_add", "ring_mul", "ring_pow",
    "ring_sub", "root_of_level", "tft", "zeros", "__version__",
]
