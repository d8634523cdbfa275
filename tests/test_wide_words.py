"""The arithmetic model behind the F32 register rounds (csrc/field.cuh F32W,
DESIGN.md §5): for a modulus 2^31 < p < 2^32, "wide" words -- any 32-bit value
congruent to the residue -- are closed under the butterfly's sum and
difference when the other operand is canonical, and the Montgomery product
takes any 32-bit multiplicand to a canonical word.  A numpy restatement of
the device formulas on random and edge values; the device code itself is
checked by tools/cu/f32wide.cu, the ring-creation probe and the GPU parity
tests."""

import numpy as np

P = 3221225473  # 3 * 2^30 + 1, BASELINE config 3's resolution
M32 = (1 << 32) - 1


def addw(a, b):  # a wide, b canonical
    s = a + b
    return np.where(s > M32, (s & M32) + (1 << 32) - P, s) & M32


def subw(a, b):
    return np.where(a < b, a + (1 << 32) - b + P, a - b) & M32


def mulw(y, wR, wRp):  # hi(y wR) - hi((y wRp mod 2^32) p), + p on borrow
    hi = (y * wR) >> 32
    m = (y * wRp) & M32
    u = (m * P) >> 32
    return np.where(hi < u, hi + P - u, hi - u)


def values(rng, n):
    edge = np.array([0, 1, P - 1, P, P + 1, M32, 1 << 31, (1 << 30) - 1, 1 << 30], dtype=object)
    return np.concatenate([edge, rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(object)])


def test_wide_sum_and_difference_stay_wide_and_congruent():
    rng = np.random.default_rng(5)
    a = values(rng, 4000)
    b = np.concatenate([np.array([0, 1, P - 1, P >> 1], dtype=object),
                        rng.integers(0, P, len(a) - 4, dtype=np.uint64).astype(object)])
    s, d = addw(a, b), subw(a, b)
    assert all(0 <= int(v) <= M32 for v in s) and all(0 <= int(v) <= M32 for v in d)
    assert all((int(x) - int(y) - int(z)) % P == 0 for x, y, z in zip(s, a, b))
    assert all((int(x) - int(y) + int(z)) % P == 0 for x, y, z in zip(d, a, b))


def test_montgomery_product_of_a_wide_word_is_canonical():
    rng = np.random.default_rng(6)
    y = values(rng, 4000)
    w = rng.integers(0, P, len(y), dtype=np.uint64).astype(object)
    pinv = pow(P, -1, 1 << 32)
    wR = np.array([(int(v) << 32) % P for v in w], dtype=object)
    wRp = np.array([(int(v) * pinv) & M32 for v in wR], dtype=object)
    r = mulw(y, wR, wRp)
    assert all(0 <= int(v) < P for v in r)
    assert all((int(v) - int(a) * int(b)) % P == 0 for v, a, b in zip(r, y, w))


def test_narrow_is_the_canonical_residue():
    rng = np.random.default_rng(7)
    x = values(rng, 2000)
    nar = np.array([min(int(v), (int(v) - P) & M32) for v in x], dtype=object)
    assert all(int(a) == int(b) % P for a, b in zip(nar, x))
