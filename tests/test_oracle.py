"""The oracle (oracle/tft_oracle.c) pinned against vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import gen, sha
from oracle import oracle as O


@pytest.fixture(scope="module")
def primes(golden):
    return {k: tuple(v) for k, v in golden["primes"].items()}


def test_known_answers(golden, primes):
    for case in golden["known"]:
        p, top, K = primes[case["prime"]]
        if case["op"] == "tft":
            assert list(O.tft(np.array(case["x"], dtype=np.uint64), p, top, K)) == case["y"]
        else:
            assert list(O.multiply(case["a"], case["b"], p, top, K)) == case["y"]


def test_config1_golden(golden, primes):
    p, top, K = primes["p998244353"]
    c1 = golden["config1"]
    y = O.tft(gen(0, p, 1000), p, top, K)
    assert sha(y) == c1["sha256_u64"] == "dbe59b5b0622d91f31c0c88b2d6feb1f5ee94677e2504dd8b48851c3076e2da3"
    assert list(y) == c1["tft"]


def test_vectors(golden, primes):
    for case in golden["vectors"]:
        p, top, K = primes[case["prime"]]
        x = gen(case["seed_x"], p, case["n"])
        y = gen(case["seed_y"], p, case["n"])
        assert list(O.tft(x, p, top, K)) == case["tft_x"], (case["prime"], case["n"])
        assert list(O.itft(y, p, top, K)) == case["itft_y"], (case["prime"], case["n"])


def test_digests(golden, primes):
    for case in golden["digests"]:
        if case["n"] > 300000:
            continue  # the big ones are pinned on the GPU path
        p, top, K = primes[case["prime"]]
        x = gen(case["seed_x"], p, case["n"])
        y = gen(case["seed_y"], p, case["n"])
        assert sha(O.tft(x, p, top, K)) == case["tft_x"], (case["prime"], case["n"])
        assert sha(O.itft(y, p, top, K)) == case["itft_y"], (case["prime"], case["n"])


def test_products(golden, primes):
    for case in golden["products"]:
        p, top, K = primes[case["prime"]]
        assert list(O.multiply(case["a"], case["b"], p, top, K)) == case["x"]
        assert list(O.schoolbook(case["a"], case["b"], p)) == case["x"]


def test_product_digests(golden, primes):
    for case in golden["product_digests"]:
        if case["la"] + case["lb"] > 200000:
            continue
        p, top, K = primes[case["prime"]]
        g = np.random.default_rng(case["seed"])
        a = g.integers(0, p, case["la"], dtype=np.uint64)
        b = g.integers(0, p, case["lb"], dtype=np.uint64)
        assert sha(O.multiply(a, b, p, top, K)) == case["x"]


def test_naive_dft_and_round_trip(primes):
    for key in ("p17", "p998244353", "p4179340454199820289"):
        p, top, K = primes[key]
        for n in range(1, min(1 << K, 70) + 1):
            x = gen(n, p, n)
            y = O.tft(x, p, top, K)
            assert np.array_equal(y, O.naive_dft(x, p, top, K))
            assert np.array_equal(O.itft(y, p, top, K), x)


def test_reference_kernels_agree_when_built(primes):
    """The reference's own compiled kernels (oracle/_ref) and the oracle give
    the same words (skipped where oracle/_ref was not built)."""
    ref = O.ref_kernels()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from array import array
    p, top, K = primes["p998244353"]
    for n in (1, 2, 3, 1000, 4097, 30001):
        x = gen(n + 7, p, n)
        buf = array("Q", x.tobytes())
        ref.tft(memoryview(buf), 0, n, p, top, K)
        assert np.array_equal(np.frombuffer(buf.tobytes(), dtype=np.uint64), O.tft(x, p, top, K))


def test_oracle_matches_reference_config5_digests():
    """The oracle against the reference's digests of config 5's pinned
    inputs (tests/golden/configs.json), the lengths it finishes quickly."""
    import json
    import os
    import workloads as W
    from conftest import sha
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "configs.json")) as f:
        cg = json.load(f)
    done = 0
    for rec in cg["config5"]:
        if rec["n"] > 20000:
            continue
        p, top, K = cg["rings"][str(rec["p"])]
        x = W.c5(rec["n"], rec["leg"], 1)
        assert sha(O.tft(x, p, top, K)) == rec["tft"][0], (rec["leg"], rec["n"])
        assert sha(O.itft(x, p, top, K)) == rec["itft"][0], (rec["leg"], rec["n"])
        done += 1
    assert done >= 30
