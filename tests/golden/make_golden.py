"""Generate tests/golden/golden.json from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    make -C oracle ref            # the reference's compiled kernels -> oracle/_ref
    python tests/golden/make_golden.py            # golden.json and tallies.json
    python tests/golden/make_golden.py --tallies  # tallies.json only

Two sources, both the reference's own code:
  * the public pure-Python API of `tftmul` imported from
    /root/reference/pkg/src (tft / itft / multiply / naive_dft), used for the
    small known-answer and cross-check cases;
  * the reference's compiled Cython kernels (`_kernels.pyx:415-480`, built
    from the reference source by oracle/Makefile), used for everything larger.
The reference test-suite asserts the two produce identical values
(`tests/test_backends.py:32-91`); this script re-asserts it on the small cases.

Inputs are regenerated from seeds with numpy's PCG64 (`default_rng(seed)
.integers(0, p, n, dtype=uint64)`, the generator BASELINE.md pins), so the
fixture stores seeds, small vectors verbatim and sha256 digests (u64
little-endian) for large outputs.  Nothing here is read at run time on the
GPU box except the JSON it writes.
"""

import hashlib
import json
import os
import sys
import time
from array import array

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import tftmul  # noqa: E402  (the reference package, pure path)
from oracle.oracle import ref_kernels  # noqa: E402

K_ = ref_kernels()
assert K_ is not None, "build the reference kernels first: make -C oracle ref"

PRIMES = {
    "p17": (17, 3, 4),
    "p998244353": (998244353, pow(3, 119, 998244353), 23),
}
for _p in (3221225473, 4179340454199820289):
    _c = tftmul.config_for_modulus(_p)
    PRIMES[f"p{_p}"] = (_c.p, _c.omegaK, _c.K)


def gen(seed, p, n):
    return np.random.default_rng(seed).integers(0, p, n, dtype=np.uint64)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def ref_tft(x, p, top, K, inverse=False):
    buf = array("Q", np.ascontiguousarray(x, dtype=np.uint64).tobytes())
    if inverse:
        K_.itft(memoryview(buf), 0, len(buf), p, top, K, (p + 1) >> 1)
    else:
        K_.tft(memoryview(buf), 0, len(buf), p, top, K)
    return np.frombuffer(buf.tobytes(), dtype=np.uint64)


def ref_mul(a, b, p, top, K):
    A = array("Q", a.tobytes())
    B = array("Q", b.tobytes())
    X = array("Q", bytes(8 * (len(A) + len(B) - 1)))
    K_.multiply(memoryview(A), memoryview(B), memoryview(X), p, top, K, (p + 1) >> 1)
    return np.frombuffer(X.tobytes(), dtype=np.uint64)


def pure_cfg(key):
    p, top, K = PRIMES[key]
    return tftmul.RingConfig(p, top, K)


def main():
    t0 = time.time()
    out = {"generator": "numpy.random.default_rng(seed).integers(0, p, n, dtype=uint64)",
           "primes": {k: list(v) for k, v in PRIMES.items()},
           "known": [], "vectors": [], "digests": [], "products": [], "product_digests": []}

    # -- known answers straight from the reference's public API ----------------
    c17 = pure_cfg("p17")
    cdef = tftmul.default_config()
    for key, cfg, data in (("p17", c17, [1, 1, 1]), ("p17", c17, [1, 2, 3, 4]),
                           ("p17", c17, [9]), ("p17", c17, [5, 3]),
                           ("p998244353", cdef, [1, 2, 3, 4])):
        buf = tftmul.make_buffer(data, cfg)
        tftmul.tft(buf, cfg)
        out["known"].append({"prime": key, "op": "tft", "x": data, "y": list(buf)})
    for key, cfg, a, b in (("p17", c17, [2, 3], [4, 5, 6]), ("p17", c17, [1, 1], [1, 1]),
                           ("p17", c17, [1], [1])):
        x = tftmul.zeros(len(a) + len(b) - 1, cfg)
        tftmul.multiply(tftmul.make_buffer(a, cfg), tftmul.make_buffer(b, cfg), x, cfg)
        out["known"].append({"prime": key, "op": "multiply", "a": a, "b": b, "y": list(x)})

    # -- verbatim vectors: tft(x) and itft(y) of independent random inputs ----
    lens_small = list(range(1, 41)) + [63, 64, 65, 100, 127, 128, 129, 255, 256, 257,
                                       777, 1000, 1023, 1024, 1025]
    seed = 1000
    for key, (p, top, K) in PRIMES.items():
        lens = [n for n in lens_small if n <= (1 << K)]
        for n in lens:
            x = gen(seed, p, n)
            y = gen(seed + 1, p, n)
            fx = ref_tft(x, p, top, K)
            iy = ref_tft(y, p, top, K, inverse=True)
            if n <= 64:
                # cross-check: the pure-Python reference path agrees
                cfg = tftmul.RingConfig(p, top, K)
                b = tftmul.make_buffer([int(v) for v in x], cfg)
                tftmul.tft(b, cfg)
                assert list(b) == [int(v) for v in fx], (key, n)
                if n <= 24:
                    assert tftmul.naive_dft([int(v) for v in x], cfg) == [int(v) for v in fx]
            out["vectors"].append({"prime": key, "n": n, "seed_x": seed, "seed_y": seed + 1,
                                   "tft_x": [int(v) for v in fx],
                                   "itft_y": [int(v) for v in iy]})
            seed += 2

    # -- digests for larger lengths (inputs regenerated from the seed) --------
    big = {
        "p998244353": [1536, 4097, 6548, 8191, 8193, 32772, 54613, 65530, 65536, 65537,
                       100003, 262145, 1000001, 4250004],
        "p3221225473": [1536, 8193, 65537, 1 << 20, (1 << 20) + 1, 3 << 19],
        "p4179340454199820289": [1536, 8193, 65537, 300001],
    }
    for key, lens in big.items():
        p, top, K = PRIMES[key]
        for n in lens:
            x = gen(seed, p, n)
            y = gen(seed + 1, p, n)
            fx = ref_tft(x, p, top, K)
            iy = ref_tft(y, p, top, K, inverse=True)
            back = ref_tft(fx, p, top, K, inverse=True)
            assert np.array_equal(back, x), (key, n)
            out["digests"].append({"prime": key, "n": n, "seed_x": seed, "seed_y": seed + 1,
                                   "tft_x": sha(fx), "itft_y": sha(iy),
                                   "tft_x_head": [int(v) for v in fx[:8]],
                                   "itft_y_head": [int(v) for v in iy[:8]]})
            seed += 2
            print(f"digest {key} n={n} ({time.time() - t0:.1f}s)", flush=True)

    # -- config 1 golden --------------------------------------
    p, top, K = PRIMES["p998244353"]
    x = gen(0, p, 1000)
    fx = ref_tft(x, p, top, K)
    out["config1"] = {"seed": 0, "n": 1000, "tft": [int(v) for v in fx], "sha256_u64": sha(fx),
                      "sha256_u32": hashlib.sha256(fx.astype("<u4").tobytes()).hexdigest()}

    # -- products ---------------------------------------------------------------
    rng = np.random.default_rng(77)
    for key in ("p17", "p998244353", "p3221225473", "p4179340454199820289"):
        p, top, K = PRIMES[key]
        shapes = [(1, 1), (1, 5), (5, 1), (2, 3), (7, 9), (16, 17), (31, 33), (64, 64),
                  (100, 29), (129, 127)]
        for la, lb in shapes:
            if la + lb - 1 > (1 << K):
                continue
            a = rng.integers(0, p, la, dtype=np.uint64)
            b = rng.integers(0, p, lb, dtype=np.uint64)
            X = ref_mul(a, b, p, top, K)
            out["products"].append({"prime": key, "a": [int(v) for v in a],
                                    "b": [int(v) for v in b], "x": [int(v) for v in X]})
    # large products by digest: inputs from a seed, A then B (BASELINE.md C4 order)
    for key, la, lb, s in (("p998244353", 5000, 3001, 501), ("p998244353", 65536, 65537, 502),
                           ("p998244353", 250001, 175004, 503),
                           ("p3221225473", 40000, 30001, 504),
                           ("p4179340454199820289", 20000, 12345, 505),
                           ("p998244353", 2500001, 1750004, 3)):
        p, top, K = PRIMES[key]
        g = np.random.default_rng(s)
        a = g.integers(0, p, la, dtype=np.uint64)
        b = g.integers(0, p, lb, dtype=np.uint64)
        X = ref_mul(a, b, p, top, K)
        out["product_digests"].append({"prime": key, "la": la, "lb": lb, "seed": s,
                                       "x": sha(X), "x_head": [int(v) for v in X[:8]],
                                       "note": "C4 first pair" if s == 3 else ""})
        print(f"product {key} {la}x{lb} ({time.time() - t0:.1f}s)", flush=True)

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"wrote golden.json in {time.time() - t0:.1f}s")


def tallies():
    """tests/golden/tallies.json: the (mults, adds) the reference's compiled
    kernels return (`_kernels.pyx:415-480`) -- value-independent, so zeros in."""
    t0 = time.time()
    out = {"transforms": [], "products": []}
    sizes = {
        "p17": list(range(1, 17)),
        "p998244353": list(range(1, 301)) + [1000, 1023, 1024, 1025, 8191, 8193, 16385, 32772, 49153,
                                             54613, 65530, 65537, 131073, 1 << 22, (1 << 22) + 1,
                                             3 << 21, (1 << 23) - 1, 1 << 23],
        "p3221225473": [1, 2, 3, 100, 65537, (1 << 20) + 1, 3 << 19],
        "p4179340454199820289": [1, 2, 3, 100, 65537, 300001],
    }
    for key, lens in sizes.items():
        p, top, K = PRIMES[key]
        for n in lens:
            z = array("Q", bytes(8 * n))
            fm, fa = K_.tft(memoryview(z), 0, n, p, top, K)
            im, ia = K_.itft(memoryview(z), 0, n, p, top, K, (p + 1) >> 1)
            out["transforms"].append({"prime": key, "n": n, "tft": [fm, fa], "itft": [im, ia]})
        print(f"tallies {key} ({time.time() - t0:.1f}s)", flush=True)
    for key, la, lb in (("p17", 1, 1), ("p17", 2, 3), ("p17", 5, 9), ("p998244353", 1, 1000),
                        ("p998244353", 64, 64), ("p998244353", 100, 29), ("p998244353", 3001, 1999),
                        ("p998244353", 65536, 65537), ("p998244353", 2500001, 1750004),
                        ("p3221225473", 40000, 30001), ("p4179340454199820289", 20000, 12345)):
        p, top, K = PRIMES[key]
        A, B = array("Q", bytes(8 * la)), array("Q", bytes(8 * lb))
        X = array("Q", bytes(8 * (la + lb - 1)))
        m, a = K_.multiply(memoryview(A), memoryview(B), memoryview(X), p, top, K, (p + 1) >> 1)
        out["products"].append({"prime": key, "la": la, "lb": lb, "tally": [m, a]})
    with open(os.path.join(HERE, "tallies.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"wrote tallies.json in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    if "--tallies" in sys.argv:
        tallies()
    else:
        main()
        tallies()
