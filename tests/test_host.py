"""Host-side logic of the package (no GPU): config validation, omega order,
schedule, buffer screening and argument errors raised before dispatch.
Mirrors the reference's tests/test_modring.py / test_polymul.py checks."""

from array import array

import numpy as np
import pytest

import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import backend
from paper_1001_5272_b200.modring import RingConfigError, UnsupportedSizeError


def small():
    return T.RingConfig(17, 3, 4)


def test_ring_config_validation():
    T.RingConfig(17, 3, 4)
    with pytest.raises(RingConfigError):
        T.RingConfig(15, 2, 1)            # not prime
    with pytest.raises(RingConfigError):
        T.RingConfig(2, 1, 0)             # even
    with pytest.raises(RingConfigError):
        T.RingConfig(17, 3, 5)            # 2^5 does not divide 16
    with pytest.raises(RingConfigError):
        T.RingConfig(17, 0, 4)            # not canonical
    with pytest.raises(RingConfigError):
        T.RingConfig(17, 2, 4)            # order 8, not 16
    with pytest.raises(RingConfigError):
        T.RingConfig(17, 5, 0)            # K=0 needs root 1
    with pytest.raises(RingConfigError):
        T.RingConfig(2**64 - 2**32 + 1, 7, 32)  # > 62 bits (reference modring.py:88-89)


def test_default_and_discovered_configs():
    c = T.default_config()
    assert (c.p, c.omegaK, c.K, c.inv2) == (998244353, 15311432, 23, 499122177)
    c = T.config_for_modulus(3221225473)
    assert (c.K, c.omegaK) == (30, 125)
    c = T.config_for_modulus(4179340454199820289)
    assert (c.K, c.omegaK) == (57, 68630377364883)
    with pytest.raises(RingConfigError):
        T.config_for_modulus(17, k=5)


def test_omega_order():
    c = small()
    assert [T.omega(s, c) for s in range(8)] == [1, 16, 13, 4, 9, 8, 15, 2]
    assert [T.root_of_level(k, c) for k in range(5)] == [1, 16, 13, 9, 3]
    with pytest.raises(UnsupportedSizeError):
        T.omega(16, c)


def test_revbin():
    assert T.revbin(0b0011, 4) == 0b1100
    assert T.revbin_increment(0b000, 3) == 0b100
    assert T.revbin_increment(0b100, 3) == 0b010


def test_block_schedule():
    for r in range(2, 300):
        q = 0
        for s in T.block_schedule(r):
            assert s.q == q and s.q % s.L == 0 and 2 * s.L <= r - s.q < 4 * s.L
            q += s.L
        assert q == r - 1
    assert [tuple(s) for s in T.block_schedule(4250004)][:3] == [(0, 21, 2097152), (2097152, 20, 1048576),
                                                                  (3145728, 19, 524288)]


def test_kernel_view_screening():
    assert backend.kernel_view(array("Q", [1, 2])) is not None
    assert backend.kernel_view(np.zeros(3, dtype=np.uint64)) is not None  # numpy accepted directly
    assert backend.kernel_view([1, 2, 3]) is None
    assert backend.kernel_view(array("I", [1, 2])) is None
    assert backend.kernel_view(np.zeros((2, 2), dtype=np.uint64)) is None
    ro = memoryview(array("Q", [1, 2])).toreadonly()
    assert backend.kernel_view(ro) is None
    assert backend.kernel_view(ro, writable=False) is not None


def test_argument_errors_before_dispatch():
    c = small()
    with pytest.raises(ValueError):
        T.tft(T.zeros(0, c), c)
    with pytest.raises(UnsupportedSizeError):
        T.tft(T.zeros(17, c), c)
    with pytest.raises(UnsupportedSizeError):
        T.itft(T.zeros(17, c), c)
    with pytest.raises(ValueError):
        T.fft_pow2(T.make_buffer([1, 2, 3], c), c)
    a, b = T.make_buffer([1, 2], c), T.make_buffer([3], c)
    with pytest.raises(ValueError):
        T.multiply(T.make_buffer([], c), b, T.zeros(0, c), c)
    with pytest.raises(ValueError):
        T.multiply(a, b, T.zeros(5, c), c)
    with pytest.raises(ValueError):
        T.multiply(a, b, a, c)
    big = T.make_buffer([1] * 10, c)
    with pytest.raises(UnsupportedSizeError):
        T.multiply(big, big, T.zeros(19, c), c)
    with pytest.raises(NotImplementedError):
        T.tft(T.make_buffer([1, 2], c), c, trace=[])
    with pytest.raises(ValueError):
        T.make_buffer([17], c)


def test_no_cpu_fallback_env(tmp_path):
    import subprocess
    import sys
    code = "import paper_1001_5272_b200"
    env = dict(__import__("os").environ, TFTMUL_BACKEND="pure")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=str(__import__("pathlib").Path(__file__).parent.parent))
    assert r.returncode != 0 and "no CPU path" in r.stderr


class _Len:
    """A buffer stand-in with only a length: the size checks run before
    anything touches the words."""

    def __init__(self, n):
        self.n = n

    def __len__(self):
        return self.n


def test_lengths_beyond_the_device_plans_raise_unsupported():
    """Lengths the reference's ring accepts (K = 30 for 3221225473) but the
    device plans do not cover (> 2^28 + 4) raise the reference's
    UnsupportedSizeError before any dispatch."""
    c = T.config_for_modulus(3221225473)
    for n in ((1 << 28) + 5, (1 << 29) + 1, 1 << 30):
        with pytest.raises(UnsupportedSizeError):
            T.tft(_Len(n), c)
        with pytest.raises(UnsupportedSizeError):
            T.itft(_Len(n), c)
    with pytest.raises(UnsupportedSizeError):
        T.multiply(_Len(1 << 27), _Len((1 << 27) + 100), _Len((1 << 28) + 99), c)
    from paper_1001_5272_b200.transforms import device_supports
    assert device_supports(1 << 28) and device_supports((1 << 28) + 4)
    assert not device_supports((1 << 28) + 5)
