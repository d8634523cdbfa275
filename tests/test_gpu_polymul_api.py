"""The reference polymul module's Algorithm-3 helpers on the GPU:
horner_eval (reference polymul.py:39-52) and fold_twist (:55-88), checked
the way the reference's own tests check them (tests/test_polymul.py:96-132:
plain fold, twisted fold, fold-then-transform lands on the global
evaluation points) plus exact evaluation against Python integers."""

import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_1001_5272_b200 as T  # noqa: E402


def small():
    return T.RingConfig(17, 3, 4)


def py_eval(coeffs, x, p):
    acc = 0
    for c in reversed(coeffs):
        acc = (acc * x + c) % p
    return acc


def test_fold_twist_plain_fold():
    cfg = small()
    src = T.make_buffer([1, 2, 3, 4, 5, 6, 7], cfg)
    X = T.zeros(8, cfg)
    T.fold_twist(src, X, 2, 4, 0, cfg)
    assert list(X) == [0, 0, 1 + 5, 2 + 6, 3 + 7, 4, 0, 0]


def test_fold_twist_twisted_fold_and_tallies():
    cfg = T.RingConfig(17, 3, 4, counters=T.OpCounters())
    vals = [3, 1, 4, 1, 5]
    X = T.zeros(4, cfg)
    T.fold_twist(T.make_buffer(vals, cfg), X, 0, 2, 2, cfg)
    w = T.omega(2, small())
    want = [0, 0]
    for i, v in enumerate(vals):
        want[i % 2] = (want[i % 2] + v * pow(w, i, 17)) % 17
    assert list(X)[:2] == want
    # the reference's own tallies for this call (2 per term after the first
    # plus omega(q)'s 2; 1 add per term), measured on tftmul 0.1.0
    assert (cfg.counters.mults, cfg.counters.adds) == (10, 5)


def test_fold_twist_then_transform_hits_global_points():
    cfg = T.default_config()
    rng = random.Random(7)
    for L, q, la in ((4, 4, 11), (8, 8, 20), (2, 6, 9), (4, 12, 16), (1024, 1024, 5000), (4096, 8192, 10001)):
        a = [rng.randrange(cfg.p) for _ in range(la)]
        X = T.zeros(q + L, cfg)
        T.fold_twist(T.make_buffer(a, cfg), X, q, L, q, cfg)
        block = T.make_buffer(list(X)[q:q + L], cfg)
        T.tft(block, cfg)
        for s in range(q, q + L, max(1, L // 16)):
            assert block[s - q] == py_eval(a, T.omega(s, cfg), cfg.p), (L, q, s)


def test_horner_eval_matches_python_integers():
    for cfg in (small(), T.default_config(), T.config_for_modulus(3221225473),
                T.config_for_modulus(4179340454199820289)):
        rng = random.Random(cfg.p)
        for n in (1, 2, 3, 17, 1000, 65537, 300001):
            if cfg.p == 17 and n > 1000:
                continue
            coeffs = [rng.randrange(cfg.p) for _ in range(n)]
            x = rng.randrange(cfg.p)
            assert T.horner_eval(T.make_buffer(coeffs, cfg), x, cfg) == py_eval(coeffs, x, cfg.p), (cfg.p, n)
            assert T.horner_eval(np.array(coeffs, dtype=np.uint64), x, cfg) == py_eval(coeffs, x, cfg.p)
    with pytest.raises(ValueError):
        T.horner_eval([], 3, small())


def test_last_slot_of_the_product_is_the_product_of_evaluations():
    """The reference's last product slot (polymul.py:106-107): A(w)B(w) at
    w = omega(r-1) equals the product's own last output of TFT_r."""
    cfg = T.default_config()
    rng = np.random.default_rng(3)
    a = rng.integers(0, cfg.p, 3001, dtype=np.uint64)
    b = rng.integers(0, cfg.p, 1999, dtype=np.uint64)
    r = a.size + b.size - 1
    x = np.zeros(r, dtype=np.uint64)
    T.multiply(a, b, x, cfg)
    w = T.omega(r - 1, cfg)
    T.tft(x, cfg)
    assert int(x[r - 1]) == T.horner_eval(a, w, cfg) * T.horner_eval(b, w, cfg) % cfg.p
