"""Ring configuration and scalar helpers (host side, no device work).

Mirrors the reference's `tftmul.modring` surface that the hot path touches
(reference pkg/src/tftmul/modring.py): the RingConfig invariants and error
types (:75-107), default_config (:110-113), config_for_modulus (:116-134),
omega(s) and its bit-reversed ordering (:223-234), and the array('Q') buffer
factories (:408-432).  Scalar ring ops are provided for callers that
compose with the transforms; the transforms themselves never run here.
"""

from array import array


class RingConfigError(ValueError):
    """The (p, root, K) triple does not describe a usable prime field."""


class UnsupportedSizeError(ValueError):
    """Length or level beyond what the config's 2^K roots support."""


# deterministic for every 64-bit n (first 12 primes as Miller-Rabin bases)
_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_probable_prime(n):
    if n < 2:
        return False
    for b in _BASES:
        if n % b == 0:
            return n == b
    d, s = n - 1, 0
    while not d & 1:
        d >>= 1
        s += 1
    for b in _BASES:
        y = pow(b, d, n)
        if y in (1, n - 1):
            continue
        for _ in range(s - 1):
            y = y * y % n
            if y == n - 1:
                break
        else:
            return False
    return True


def ceil_lg(n):
    """Smallest k with 2^k >= n (n >= 1)."""
    if n < 1:
        raise ValueError("ceil_lg needs n >= 1")
    return (n - 1).bit_length()


class OpCounters:
    """Operation tallies credited by the transforms (the
    device path credits its own op model, not the reference's walk)."""

    __slots__ = ("mults", "adds", "allocs")

    def __init__(self):
        self.reset()

    def reset(self):
        self.mults = 0
        self.adds = 0
        self.allocs = 0

    def __repr__(self):
        return f"OpCounters(mults={self.mults}, adds={self.adds}, allocs={self.allocs})"


class RingConfig:
    """Modulus p, a root omegaK of exact order 2^K, K and inv2 = (p+1)/2.

    Same checks, same order and same exception types as the reference
    (modring.py:85-104)."""

    __slots__ = ("p", "K", "omegaK", "inv2", "counters")

    def __init__(self, p, omegaK, K, counters=None):
        if p < 3 or p % 2 == 0 or not is_probable_prime(p):
            raise RingConfigError(f"modulus {p} is not an odd prime")
        if p >= 1 << 62:
            raise RingConfigError("modulus must fit in 62 bits")
        if K < 0 or (p - 1) % (1 << K):
            raise RingConfigError(f"2^{K} does not divide p - 1 = {p - 1}")
        if not 0 < omegaK < p:
            raise RingConfigError(f"root {omegaK} is not a canonical residue mod {p}")
        if pow(omegaK, 1 << K, p) != 1:
            raise RingConfigError(f"{omegaK} is not a 2^{K}-th root of unity mod {p}")
        if K >= 1 and pow(omegaK, 1 << (K - 1), p) != p - 1:
            raise RingConfigError(f"{omegaK} has order smaller than 2^{K} mod {p}")
        if K == 0 and omegaK != 1:
            raise RingConfigError("a 2^0-th root of unity must be 1")
        self.p = p
        self.K = K
        self.omegaK = omegaK
        self.inv2 = (p + 1) >> 1
        self.counters = counters

    def __repr__(self):
        return f"RingConfig(p={self.p}, omegaK={self.omegaK}, K={self.K})"


def default_config(instrument=False):
    """p = 119*2^23 + 1 with omegaK = 3^119 (K = 23), as the reference."""
    p = 998244353
    return RingConfig(p, pow(3, 119, p), 23, OpCounters() if instrument else None)


def config_for_modulus(p, root=None, k=None, instrument=False):
    """Config for any odd prime: K defaults to v2(p-1); without a root the
    smallest quadratic non-residue g gives root = g^((p-1)/2^k)."""
    if p < 3 or p % 2 == 0 or not is_probable_prime(p):
        raise RingConfigError(f"modulus {p} is not an odd prime")
    v2 = ((p - 1) & -(p - 1)).bit_length() - 1
    if k is None:
        k = v2
    if k > v2:
        raise RingConfigError(f"2^{k} does not divide p - 1 = {p - 1}")
    if root is None:
        g = 2
        while pow(g, (p - 1) >> 1, p) != p - 1:
            g += 1
        root = pow(g, (p - 1) >> k, p)
    return RingConfig(p, root, k, OpCounters() if instrument else None)


def _count(cfg, mults=0, adds=0):
    c = cfg.counters
    if c is not None:
        c.mults += mults
        c.adds += adds


def ring_add(a, b, cfg):
    _count(cfg, adds=1)
    s = a + b
    return s - cfg.p if s >= cfg.p else s


def ring_sub(a, b, cfg):
    _count(cfg, adds=1)
    d = a - b
    return d + cfg.p if d < 0 else d


def ring_mul(a, b, cfg):
    _count(cfg, mults=1)
    return a * b % cfg.p


def ring_pow(a, e, cfg):
    """a^e by left-to-right square and multiply; a^0 = 1."""
    if e < 0:
        raise ValueError("exponent must be nonnegative")
    if e == 0:
        return 1
    r, m = a, 0
    for i in range(e.bit_length() - 2, -1, -1):
        r = r * r % cfg.p
        m += 1
        if (e >> i) & 1:
            r = r * a % cfg.p
            m += 1
    _count(cfg, mults=m)
    return r


def root_of_level(k, cfg):
    """omega_[k] = omegaK^(2^(K-k))."""
    if not 0 <= k <= cfg.K:
        raise UnsupportedSizeError(f"level {k} outside [0, {cfg.K}]")
    _count(cfg, mults=cfg.K - k)
    return pow(cfg.omegaK, 1 << (cfg.K - k), cfg.p)


def revbin(s, k):
    """Reverse the low k bits of s (s < 2^k)."""
    if s >> k:
        raise ValueError(f"{s} does not fit in {k} bits")
    return int(format(s, f"0{k}b")[::-1], 2) if k else 0


def revbin_increment(c, k):
    """rev_k(t) -> rev_k(t+1): carries run from the top bit down."""
    if k < 1:
        raise ValueError("counter width must be at least 1")
    bit = 1 << (k - 1)
    while c & bit:
        c ^= bit
        bit >>= 1
        if not bit:
            raise ValueError("reversed counter overflow")
    return c | bit


def omega(s, cfg):
    """Evaluation point of output slot s: omega_[bitlen s]^rev(s); size
    independent."""
    if not 0 <= s < 1 << cfg.K:
        raise UnsupportedSizeError(f"index {s} outside [0, 2^{cfg.K})")
    if s == 0:
        return 1
    k = s.bit_length()
    return ring_pow(root_of_level(k, cfg), revbin(s, k), cfg)


def make_buffer(values, cfg):
    """array('Q') of canonical residues (counted as one allocation)."""
    c = cfg.counters
    if c is not None:
        c.allocs += 1
    buf = array("Q", values)
    for v in buf:
        if v >= cfg.p:
            raise ValueError(f"value {v} is not canonical mod {cfg.p}")
    return buf


def zeros(n, cfg):
    if n < 0:
        raise ValueError("length must be nonnegative")
    c = cfg.counters
    if c is not None:
        c.allocs += 1
    return array("Q", bytes(8 * n))
