"""Pinned synthetic inputs for the five BASELINE configs (BASELINE.json
`configs`).  One generator everywhere -- bench.py, the GPU
parity tests and tests/golden/make_config_golden.py (which feeds the same
words to the reference) -- so device results and reference digests are
comparable bit for bit:

    rng = numpy.random.default_rng(seed); rng.integers(0, p, size, dtype=uint64)

Residues are uniform over the whole of [0, p) (for p = 3221225473 that
includes the top quarter above 2^31, which drives the canonical-add carry
paths).  numpy's bounded generator consumes its stream sequentially, so the
first n words of a larger draw equal a draw of n words; the tests rely on
that to check the head vectors of a config-5 launch.
"""

import numpy as np

P_DEFAULT = 998244353           # default ring, K = 23
P_C3 = 3221225473               # 3 * 2^30 + 1, K = 30: config 3 / config 5 above 2^23
P_U64 = 4179340454199820289     # 29 * 2^57 + 1, K = 57: config 5's 64-bit leg

C3_LENGTHS = (1 << 24, (1 << 24) + 1, 3 << 23, (1 << 25) - 1, (1 << 25) + 1)
# the same shape at the default prime's own range (K = 23), BASELINE.md §3
C3_DEFAULT_LENGTHS = (1 << 22, (1 << 22) + 1, 3 << 21, (1 << 23) - 1, 1 << 23)
C4_LA, C4_LB, C4_PAIRS = 2500001, 1750004, 256


def words(seed, p, n):
    return np.random.default_rng(seed).integers(0, p, n, dtype=np.uint64)


def c1():
    """Config 1: n = 1000 at p = 998244353, seed 0."""
    return words(0, P_DEFAULT, 1000)


def c2_lengths(seed=1):
    rng = np.random.default_rng(seed)
    return rng.integers(2 ** 15 + 1, 2 ** 16 + 1, 4096).astype(np.int64)


def c2(seed=1):
    """Config 2: 4096 lengths uniform in [2^15+1, 2^16], then the flat words
    (one stream, seed 1).  Returns (lengths int64, flat uint64)."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(2 ** 15 + 1, 2 ** 16 + 1, 4096)
    flat = rng.integers(0, P_DEFAULT, int(lens.sum()), dtype=np.uint64)
    return lens.astype(np.int64), flat


def c3(n, p=P_C3):
    """Config 3: one vector of length n, seed 2 (each length drawn afresh)."""
    return words(2, p, n)


def c4_pairs(indices, p=P_DEFAULT):
    """Config 4: pairs drawn in order from one seed-3 stream, A (2,500,001
    words) then B (1,750,004 words) per pair.  Yields (index, a, b) for the
    requested pair indices (the stream is consumed up to the largest)."""
    want = set(int(i) for i in indices)
    rng = np.random.default_rng(3)
    for k in range(max(want) + 1):
        a = rng.integers(0, p, C4_LA, dtype=np.uint64)
        b = rng.integers(0, p, C4_LB, dtype=np.uint64)
        if k in want:
            yield k, a, b


def c4_all(p=P_DEFAULT, pairs=C4_PAIRS):
    """All pairs as two flat arrays (pairs*la, pairs*lb)."""
    rng = np.random.default_rng(3)
    A = np.empty(pairs * C4_LA, dtype=np.uint64)
    B = np.empty(pairs * C4_LB, dtype=np.uint64)
    for k in range(pairs):
        A[k * C4_LA:(k + 1) * C4_LA] = rng.integers(0, p, C4_LA, dtype=np.uint64)
        B[k * C4_LB:(k + 1) * C4_LB] = rng.integers(0, p, C4_LB, dtype=np.uint64)
    return A, B


def c5_lengths():
    """Config 5: 64 log-spaced lengths 2^10+3 .. 2^28-5, nudged off powers
    of two."""
    ns = np.round(np.geomspace(1027, 268435451, 64)).astype(np.int64)
    return [int(n) + 1 if n & (n - 1) == 0 else int(n) for n in ns]


def c5_prime(n, leg):
    """u32 leg: 998244353 up to its K = 23, 3221225473 above; u64 leg: the
    62-bit prime."""
    if leg == "u64":
        return P_U64
    return P_DEFAULT if n <= (1 << 23) else P_C3


def c5_batch(n, word_bytes=4, cap_bytes=6e9):
    """floor(2^28 / n) vectors per launch, capped by device bytes."""
    b = max(1, (1 << 28) // n)
    if b * n * word_bytes > cap_bytes:
        b = max(1, int(cap_bytes // (n * word_bytes)))
    return b


def c5(n, leg, count):
    """The first `count` vectors of config 5's launch at length n (seed 4)."""
    return words(4, c5_prime(n, leg), count * n)
