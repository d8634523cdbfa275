"""GPU parity: the CUDA path (through the C ABI) against vectors the
reference itself produced (tests/golden) and against the oracle, bit-exact.
Runs on a B200 (`pytest -m gpu`)."""

from array import array

import numpy as np
import pytest

from conftest import gen, sha

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_1001_5272_b200 as T  # noqa: E402
from paper_1001_5272_b200 import backend, device  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker only)


def cfg_for(golden, key):
    p, top, K = golden["primes"][key]
    return T.RingConfig(p, top, K)


def run(fn, x, cfg):
    buf = array("Q", np.ascontiguousarray(x, dtype=np.uint64).tobytes())
    fn(buf, cfg)
    return np.frombuffer(buf.tobytes(), dtype=np.uint64)


def test_known_answers(golden):
    for case in golden["known"]:
        cfg = cfg_for(golden, case["prime"])
        if case["op"] == "tft":
            buf = T.make_buffer(case["x"], cfg)
            T.tft(buf, cfg)
            assert list(buf) == case["y"]
            T.itft(buf, cfg)
            assert list(buf) == case["x"]
        else:
            x = T.zeros(len(case["a"]) + len(case["b"]) - 1, cfg)
            T.multiply(T.make_buffer(case["a"], cfg), T.make_buffer(case["b"], cfg), x, cfg)
            assert list(x) == case["y"]


def test_config1(golden):
    cfg = T.default_config()
    x = gen(0, cfg.p, 1000)
    y = run(T.tft, x, cfg)
    assert sha(y) == golden["config1"]["sha256_u64"]
    assert np.array_equal(run(T.itft, y, cfg), x)


def test_vectors(golden):
    for case in golden["vectors"]:
        cfg = cfg_for(golden, case["prime"])
        x = gen(case["seed_x"], cfg.p, case["n"])
        y = gen(case["seed_y"], cfg.p, case["n"])
        assert list(run(T.tft, x, cfg)) == case["tft_x"], (case["prime"], case["n"])
        assert list(run(T.itft, y, cfg)) == case["itft_y"], (case["prime"], case["n"])


def test_digests(golden):
    for case in golden["digests"]:
        cfg = cfg_for(golden, case["prime"])
        x = gen(case["seed_x"], cfg.p, case["n"])
        y = gen(case["seed_y"], cfg.p, case["n"])
        fx = run(T.tft, x, cfg)
        assert sha(fx) == case["tft_x"], ("tft", case["prime"], case["n"], list(fx[:4]), case["tft_x_head"][:4])
        iy = run(T.itft, y, cfg)
        assert sha(iy) == case["itft_y"], ("itft", case["prime"], case["n"], list(iy[:4]),
                                           case["itft_y_head"][:4])
        assert np.array_equal(run(T.itft, fx, cfg), x)


def test_products(golden):
    for case in golden["products"]:
        cfg = cfg_for(golden, case["prime"])
        a = T.make_buffer(case["a"], cfg)
        b = T.make_buffer(case["b"], cfg)
        keep = (a.tobytes(), b.tobytes())
        x = T.zeros(len(a) + len(b) - 1, cfg)
        T.multiply(a, b, x, cfg)
        assert list(x) == case["x"]
        assert (a.tobytes(), b.tobytes()) == keep


def test_product_digests(golden):
    for case in golden["product_digests"]:
        cfg = cfg_for(golden, case["prime"])
        g = np.random.default_rng(case["seed"])
        a = g.integers(0, cfg.p, case["la"], dtype=np.uint64)
        b = g.integers(0, cfg.p, case["lb"], dtype=np.uint64)
        x = np.zeros(case["la"] + case["lb"] - 1, dtype=np.uint64)
        T.multiply(a, b, x, cfg)
        assert sha(x) == case["x"], (case, list(x[:4]))


@pytest.mark.parametrize("key", ["p998244353", "p3221225473", "p4179340454199820289", "p17"])
def test_every_small_length_against_oracle(golden, key):
    cfg = cfg_for(golden, key)
    top = min(1 << cfg.K, 600)
    for n in range(1, top + 1):
        x = gen(10_000 + n, cfg.p, n)
        y = run(T.tft, x, cfg)
        assert np.array_equal(y, O.tft(x, cfg.p, cfg.omegaK, cfg.K)), n
        assert np.array_equal(run(T.itft, y, cfg), x), n


def test_two_pass_boundaries_against_oracle():
    cfg = T.default_config()
    lens = [8191, 8192, 8193, 12289, 16383, 16384, 16385, 32767, 32769, 49153, 65535, 65536, 65537,
            131071, 131073, 196609, 262143, 262145, 524287, 524289, 1048575, 1048577]
    for n in lens:
        x = gen(n, cfg.p, n)
        y = run(T.tft, x, cfg)
        assert np.array_equal(y, O.tft(x, cfg.p, cfg.omegaK, cfg.K)), n
        z = gen(n + 1, cfg.p, n)
        assert np.array_equal(run(T.itft, z, cfg), O.itft(z, cfg.p, cfg.omegaK, cfg.K)), n


def test_fft_pow2_matches_tft():
    cfg = T.default_config()
    for k in range(0, 16):
        x = gen(k, cfg.p, 1 << k)
        a = run(T.fft_pow2, x, cfg)
        assert np.array_equal(a, run(T.tft, x, cfg))


def test_maximum_size_small_ring():
    cfg = T.RingConfig(17, 3, 4)
    x = gen(5, 17, 16)
    y = run(T.tft, x, cfg)
    assert np.array_equal(y, O.naive_dft(x, 17, 3, 4))
    assert np.array_equal(run(T.itft, y, cfg), x)


def test_list_buffers_staged():
    cfg = T.RingConfig(17, 3, 4)
    buf = [1, 2, 3, 4]
    T.tft(buf, cfg)
    assert buf == [10, 15, 6, 7]


def test_device_ragged_batch_against_oracle():
    cfg = T.default_config()
    rng = np.random.default_rng(1)
    lens = rng.integers(1, 70000, 24)
    lens[:4] = [1, 2, 8192, 65536]
    flat = rng.integers(0, cfg.p, int(lens.sum()), dtype=np.uint64)
    d = device.to_words(flat, cfg)
    device.tft_batch_(d, cfg, lengths=lens)
    got = device.from_words(d, cfg)
    want = O.tft_batch(flat, lens, cfg.p, cfg.omegaK, cfg.K)
    assert np.array_equal(got, want)
    device.tft_batch_(d, cfg, lengths=lens, inverse=True)
    assert np.array_equal(device.from_words(d, cfg), flat)


def test_device_uniform_batch_and_products():
    cfg = T.default_config()
    rng = np.random.default_rng(2)
    for n in (1000, 40000):
        flat = rng.integers(0, cfg.p, 8 * n, dtype=np.uint64)
        d = device.to_words(flat, cfg)
        device.tft_batch_(d, cfg, n=n, count=8)
        want = O.tft_batch(flat, np.full(8, n), cfg.p, cfg.omegaK, cfg.K)
        assert np.array_equal(device.from_words(d, cfg), want)
    la, lb, cnt = 3001, 1999, 5
    a = rng.integers(0, cfg.p, cnt * la, dtype=np.uint64)
    b = rng.integers(0, cfg.p, cnt * lb, dtype=np.uint64)
    x = torch.zeros(cnt * (la + lb - 1), dtype=device.word_dtype(cfg), device="cuda")
    device.multiply_batch(device.to_words(a, cfg), device.to_words(b, cfg), x, cfg, cnt, la, lb)
    got = device.from_words(x, cfg).reshape(cnt, -1)
    for v in range(cnt):
        assert np.array_equal(got[v], O.multiply(a[v * la:(v + 1) * la], b[v * lb:(v + 1) * lb],
                                                 cfg.p, cfg.omegaK, cfg.K))


def test_launches_counted():
    cfg = T.default_config()
    backend.launch_count(reset=True)
    run(T.tft, gen(3, cfg.p, 5000), cfg)
    assert backend.launch_count() >= 1


def test_batch_plan_reuse_against_oracle():
    cfg = T.default_config()
    rng = np.random.default_rng(11)
    lens = rng.integers(1, 140000, 40)
    lens[:6] = [1, 16384, 16385, 32768, 49153, 131072]
    flat = rng.integers(0, cfg.p, int(lens.sum()), dtype=np.uint64)
    plan = device.BatchPlan(cfg, lens)
    d = device.to_words(flat, cfg)
    want = O.tft_batch(flat, lens, cfg.p, cfg.omegaK, cfg.K)
    for _ in range(2):
        plan.execute(d)
        assert np.array_equal(device.from_words(d, cfg), want)
        plan.execute(d, inverse=True)
        assert np.array_equal(device.from_words(d, cfg), flat)


def test_tile_plain_inverse_every_size():
    """Regression: the unmasked in-tile inverse (two-pass chunk step) at every
    tile size, through the internal debug entry point."""
    import ctypes
    cfg = T.default_config()
    lib = backend.load()
    f = lib.tftb_debug_intt_tile
    f.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    for t in range(1, 15):
        y = gen(t, cfg.p, 1 << t)
        d = device.to_words(y, cfg)
        backend.check(f(cfg.p, cfg.omegaK, cfg.K, d.data_ptr(), t))
        assert np.array_equal(device.from_words(d, cfg), O.itft(y, cfg.p, cfg.omegaK, cfg.K)), t


def test_host_batch_pipeline_against_oracle():
    """tftb_tft_batch_u64 (pipelined host batch) on a ragged batch, both directions."""
    import ctypes
    cfg = T.default_config()
    rng = np.random.default_rng(21)
    lens = rng.integers(1, 90000, 300).astype(np.int64)
    flat = rng.integers(0, cfg.p, int(lens.sum()), dtype=np.uint64)
    x = flat.copy()
    lib = backend.load()
    lp = lens.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    backend.check(lib.tftb_tft_batch_u64(x.ctypes.data, None, lp, lens.size, cfg.p, cfg.omegaK, cfg.K, 0))
    assert np.array_equal(x, O.tft_batch(flat, lens, cfg.p, cfg.omegaK, cfg.K))
    backend.check(lib.tftb_tft_batch_u64(x.ctypes.data, None, lp, lens.size, cfg.p, cfg.omegaK, cfg.K, 1))
    assert np.array_equal(x, flat)


@pytest.mark.parametrize("key", ["p998244353", "p3221225473", "p4179340454199820289"])
def test_shared_cta_small_tiles_against_oracle(golden, key):
    """Many short vectors of one size class share a CTA (k_tile_*): ragged
    lengths inside each class, partly-filled last CTA, both directions."""
    cfg = cfg_for(golden, key)
    rng = np.random.default_rng(31)
    lens = np.concatenate([rng.integers(1, 33, 300), rng.integers(33, 257, 300),
                           rng.integers(257, 4097, 61), [1, 2, 3, 32, 33, 4096]])
    rng.shuffle(lens)
    flat = rng.integers(0, cfg.p, int(lens.sum()), dtype=np.uint64)
    d = device.to_words(flat, cfg)
    device.tft_batch_(d, cfg, lengths=lens)
    assert np.array_equal(device.from_words(d, cfg), O.tft_batch(flat, lens, cfg.p, cfg.omegaK, cfg.K))
    device.tft_batch_(d, cfg, lengths=lens, inverse=True)
    assert np.array_equal(device.from_words(d, cfg), flat)
    for la, lb, cnt in ((7, 5, 33), (100, 29, 9)):
        a = rng.integers(0, cfg.p, cnt * la, dtype=np.uint64)
        b = rng.integers(0, cfg.p, cnt * lb, dtype=np.uint64)
        x = torch.zeros(cnt * (la + lb - 1), dtype=device.word_dtype(cfg), device="cuda")
        device.multiply_batch(device.to_words(a, cfg), device.to_words(b, cfg), x, cfg, cnt, la, lb)
        got = device.from_words(x, cfg).reshape(cnt, -1)
        for v in range(cnt):
            assert np.array_equal(got[v], O.multiply(a[v * la:(v + 1) * la], b[v * lb:(v + 1) * lb],
                                                     cfg.p, cfg.omegaK, cfg.K)), (la, lb, v)


def test_host_api_returns_reference_tallies(golden):
    """_kernels-shaped calls return the reference walk's (mults, adds)."""
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "tallies.json")) as f:
        tallies = json.load(f)
    k = backend.kernels()
    for case in tallies["transforms"][::7]:
        p, top, K = golden["primes"][case["prime"]]
        if case["n"] > (1 << 20):
            continue
        x = array("Q", bytes(8 * case["n"]))
        assert list(k.tft(x, 0, case["n"], p, top, K)) == case["tft"]
        assert list(k.itft(x, 0, case["n"], p, top, K, (p + 1) // 2)) == case["itft"]
    for case in tallies["products"]:
        p, top, K = golden["primes"][case["prime"]]
        if case["la"] + case["lb"] > 200000:
            continue
        a, b = array("Q", bytes(8 * case["la"])), array("Q", bytes(8 * case["lb"]))
        x = array("Q", bytes(8 * (case["la"] + case["lb"] - 1)))
        assert list(k.multiply(a, b, x, p, top, K, (p + 1) // 2)) == case["tally"]


@pytest.mark.parametrize("key", ["p998244353", "p3221225473", "p4179340454199820289"])
def test_power_of_two_plus_r_against_oracle(golden, key):
    """n = 2^k + r, r <= 4, beyond the cluster range: the 2^k transform plus r
    dot products (p2r.cuh) -- both directions, single and batched."""
    cfg = cfg_for(golden, key)
    for n in [(1 << 18) + r for r in (1, 2, 3, 4)] + [(1 << 19) + 4, (1 << 18) + 5]:
        x = gen(70_000 + n, cfg.p, n)
        assert np.array_equal(run(T.tft, x, cfg), O.tft(x, cfg.p, cfg.omegaK, cfg.K)), n
        z = gen(80_000 + n, cfg.p, n)
        assert np.array_equal(run(T.itft, z, cfg), O.itft(z, cfg.p, cfg.omegaK, cfg.K)), n
    n, cnt = (1 << 18) + 3, 3
    flat = gen(90_001, cfg.p, n * cnt)
    plan = device.BatchPlan(cfg, np.full(cnt, n))
    d = device.to_words(flat, cfg)
    plan.execute(d)
    assert np.array_equal(device.from_words(d, cfg), O.tft_batch(flat, np.full(cnt, n), cfg.p, cfg.omegaK, cfg.K))
    plan.execute(d, inverse=True)
    assert np.array_equal(device.from_words(d, cfg), flat)


def test_u64_past_two_to_the_26_round_trip_and_oracle_head(golden):
    """u64 words beyond 2^26 run the two-pass plan with 2^14-word tiles:
    exact round trip at 2^26 + 3 (p2r prefix) and 3 * 2^25, and the first
    outputs against the oracle's naive evaluation."""
    cfg = cfg_for(golden, "p4179340454199820289")
    for n in ((1 << 26) + 3, 3 << 25):
        flat = gen(123 + n, cfg.p, n)
        d = device.to_words(flat, cfg)
        device.tft_batch_(d, cfg, n=n)
        got = device.from_words(d, cfg)
        # outputs 0 and 1 are sum x and the alternating sum (omega_0 = 1, omega_1 = -1)
        p = cfg.p
        s0 = int(sum(int(v) for v in flat[::1]) % p)
        assert int(got[0]) == s0
        device.tft_batch_(d, cfg, n=n, inverse=True)
        assert torch.equal(d, device.to_words(flat, cfg)), n


@pytest.mark.gpu
def test_device_footprint_audit():
    """The in-place claim on device: tile and cluster plans (n <= 2^17 u32)
    allocate nothing beyond the n words; larger transforms at most a stash
    of one chunk (2^14 words) per vector plus p2r partial sums -- O(sqrt n),
    independent of n."""
    import numpy as np
    import paper_1001_5272_b200 as T
    from paper_1001_5272_b200 import backend
    cfg = T.default_config()
    for n in (16, 512, 5000, 40000, 131072):
        x = np.random.default_rng(n).integers(0, cfg.p, n, dtype=np.uint64)
        backend.aux_bytes(reset=True)
        T.tft(x, cfg)
        T.itft(x, cfg)
        assert backend.aux_bytes() == 0, n
    peaks = []
    for n in (2 ** 18 + 7, 2 ** 20 + 1, 2 ** 21 - 3, 3 * 2 ** 21):
        x = np.random.default_rng(n).integers(0, cfg.p, n, dtype=np.uint64)
        backend.aux_bytes(reset=True)
        T.tft(x, cfg)
        T.itft(x, cfg)
        peaks.append(backend.aux_bytes())
    assert max(peaks) <= 2 ** 14 * 4 + 32768, peaks  # one chunk stash + p2r partial sums


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["p998244353", "p3221225473", "p4179340454199820289"])
def test_cluster_range_every_chunk_count_against_oracle(golden, key):
    """The chunked plans (forward cone + split inverse) on every word type:
    G = 2..8 chunks, complete last chunk (h = 0) and ragged ones, in a
    ragged device batch and through the host API."""
    cfg = cfg_for(golden, key)
    C = 1 << (14 if cfg.p < 2 ** 32 else 13)
    lens = []
    for G in range(2, 9):
        lens += [G * C, (G - 1) * C + 1, (G - 1) * C + C // 2 + 3, G * C - 1]
    lens = np.array(lens, dtype=np.int64)
    rng = np.random.default_rng(77)
    flat = rng.integers(0, cfg.p, int(lens.sum()), dtype=np.uint64)
    d = device.to_words(flat, cfg)
    device.tft_batch_(d, cfg, lengths=lens)
    got = device.from_words(d, cfg)
    assert np.array_equal(got, O.tft_batch(flat, lens, cfg.p, cfg.omegaK, cfg.K))
    device.tft_batch_(d, cfg, lengths=lens, inverse=True)
    assert np.array_equal(device.from_words(d, cfg), flat)
    # inverse of arbitrary words (not a forward image) against the oracle
    z = rng.integers(0, cfg.p, int(lens[:8].sum()), dtype=np.uint64)
    dz = device.to_words(z, cfg)
    device.tft_batch_(dz, cfg, lengths=lens[:8], inverse=True)
    off = np.concatenate([[0], np.cumsum(lens[:8])])
    want = np.concatenate([O.itft(z[off[i]:off[i + 1]], cfg.p, cfg.omegaK, cfg.K) for i in range(8)])
    assert np.array_equal(device.from_words(dz, cfg), want)


@pytest.mark.gpu
def test_products_in_the_chunked_range_against_oracle():
    """Products whose length r uses the chunked plans (forward cone or split
    forward, split inverse with the pointwise factor fused into its load)."""
    cfg = T.default_config()
    for la, lb in ((10, 16400), (20000, 20001), (30000, 35537), (70000, 40000), (1, 65536)):
        a = gen(la, cfg.p, la)
        b = gen(lb + 1, cfg.p, lb)
        out = np.zeros(la + lb - 1, dtype=np.uint64)
        T.multiply(a, b, out, cfg)
        assert np.array_equal(out, O.multiply(a, b, cfg.p, cfg.omegaK, cfg.K)), (la, lb)


@pytest.mark.gpu
def test_concurrent_calls_on_distinct_buffers():
    """The reference's concurrency model: calls on distinct buffers may run
    at once (its kernels release the GIL; ctypes does too).  Several host
    threads transform, invert and multiply their own buffers together."""
    import threading
    cfg = T.default_config()
    errors = []

    def worker(k):
        try:
            for r in range(3):
                n = [1000, 40000, 70001, 2 ** 20 + 1][(k + r) % 4]
                x = gen(100 * k + r, cfg.p, n)
                y = x.copy()
                T.tft(y, cfg)
                if n <= 70001:
                    assert np.array_equal(y, O.tft(x, cfg.p, cfg.omegaK, cfg.K)), n
                T.itft(y, cfg)
                assert np.array_equal(y, x), n
                a, b = gen(k, cfg.p, 3000 + k), gen(k + 50, cfg.p, 2000)
                out = np.zeros(a.size + b.size - 1, dtype=np.uint64)
                T.multiply(a, b, out, cfg)
                assert np.array_equal(out, O.multiply(a, b, cfg.p, cfg.omegaK, cfg.K))
        except Exception as e:  # noqa: BLE001  (reported below)
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


@pytest.mark.gpu
def test_layout_validation_rejects_bad_batches():
    """Negative offsets, overlapping vectors, short strides and short
    scratch are rejected before any launch (Python wrapper and C ABI)."""
    import ctypes
    cfg = T.default_config()
    d = torch.zeros(1000, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        device.tft_batch_(d, cfg, lengths=[10, 10], offsets=[-1, 20])
    with pytest.raises(ValueError):
        device.tft_batch_(d, cfg, lengths=[10, 10], offsets=[0, 5])
    with pytest.raises(ValueError):
        device.tft_batch_(d, cfg, n=10, count=3, stride=5)
    with pytest.raises(ValueError):
        device.BatchPlan(cfg, [10, 10], [30, 25])
    a = torch.zeros(20, dtype=torch.int32, device="cuda")
    x = torch.zeros(39, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        device.multiply_batch(a, a, x, cfg, 1, 20, 20, scratch=torch.zeros(5, dtype=torch.int32, device="cuda"))
    # the C ABI itself
    lib = backend.load()
    h = backend.ring_handle(cfg)
    off = np.array([0, 5], dtype=np.int64)
    ln = np.array([10, 10], dtype=np.int64)
    p64 = ctypes.POINTER(ctypes.c_int64)
    rc = lib.tftb_tft_dev(h, ctypes.c_void_p(d.data_ptr()), 2, 0, 0, off.ctypes.data_as(p64),
                          ln.ctypes.data_as(p64), 0, None)
    assert rc != 0 and b"overlap" in lib.tftb_last_error()
    off = np.array([-3, 50], dtype=np.int64)
    rc = lib.tftb_tft_dev(h, ctypes.c_void_p(d.data_ptr()), 2, 0, 0, off.ctypes.data_as(p64),
                          ln.ctypes.data_as(p64), 0, None)
    assert rc != 0
    rc = lib.tftb_tft_dev(h, ctypes.c_void_p(d.data_ptr()), 3, 10, 5, None, None, 0, None)
    assert rc != 0


@pytest.mark.gpu
def test_host_batch_with_gaps_and_unsorted_offsets():
    """tftb_tft_batch_u64 transforms only the [off, off+len) runs: words in
    the gaps (even ones >= 2^32, which no u32 ring word can hold) come back
    untouched; unsorted offsets work; overlapping ones are rejected."""
    import ctypes
    cfg = T.default_config()
    rng = np.random.default_rng(5)
    lens = np.array([700, 40000, 1, 9000, 70001, 33], dtype=np.int64)
    gaps = np.array([3, 0, 17, 1, 5, 2], dtype=np.int64)
    offs = np.zeros_like(lens)
    pos = 0
    for i in range(lens.size):
        pos += gaps[i]
        offs[i] = pos
        pos += lens[i]
    buf = np.full(pos + 7, (1 << 40) + 12345, dtype=np.uint64)
    for o, n in zip(offs, lens):
        buf[o:o + n] = rng.integers(0, cfg.p, n, dtype=np.uint64)
    orig = buf.copy()
    perm = np.array([3, 0, 5, 1, 4, 2])
    lib = backend.load()
    p64 = ctypes.POINTER(ctypes.c_int64)
    o2, l2 = offs[perm].copy(), lens[perm].copy()
    backend.check(lib.tftb_tft_batch_u64(buf.ctypes.data, o2.ctypes.data_as(p64), l2.ctypes.data_as(p64),
                                         lens.size, cfg.p, cfg.omegaK, cfg.K, 0))
    mask = np.ones(buf.size, dtype=bool)
    for o, n in zip(offs, lens):
        mask[o:o + n] = False
        assert np.array_equal(buf[o:o + n], O.tft(orig[o:o + n], cfg.p, cfg.omegaK, cfg.K)), n
    assert np.array_equal(buf[mask], orig[mask])
    backend.check(lib.tftb_tft_batch_u64(buf.ctypes.data, o2.ctypes.data_as(p64), l2.ctypes.data_as(p64),
                                         lens.size, cfg.p, cfg.omegaK, cfg.K, 1))
    assert np.array_equal(buf, orig)
    bad = np.array([0, 500], dtype=np.int64)
    rc = lib.tftb_tft_batch_u64(buf.ctypes.data, bad.ctypes.data_as(p64), lens[:2].copy().ctypes.data_as(p64),
                                2, cfg.p, cfg.omegaK, cfg.K, 0)
    assert rc != 0 and b"overlap" in lib.tftb_last_error()


@pytest.mark.gpu
def test_host_api_device_memory_is_the_ring_words_plus_bounded_staging():
    """The host-pointer calls convert uint64 words through a bounded staging
    buffer: device memory ~ 4 B per word for u32 rings (+ 32 MB), 8 B for u64."""
    cfg = T.default_config()
    for n in (1000, 70001, 3 << 21):
        x = gen(n, cfg.p, n)
        backend.stage_bytes(reset=True)
        y = x.copy()
        T.tft(y, cfg)
        T.itft(y, cfg)
        assert np.array_equal(y, x)
        used = backend.stage_bytes()
        assert used <= 4 * n + 8 * min(n, 1 << 22) + 512, (n, used)
    a, b = gen(1, cfg.p, 1 << 20), gen(2, cfg.p, 1 << 20)
    out = np.zeros(a.size + b.size - 1, dtype=np.uint64)
    backend.stage_bytes(reset=True)
    T.multiply(a, b, out, cfg)
    r = out.size
    assert backend.stage_bytes() <= 4 * (a.size + b.size + 2 * r) + 8 * min(r, 1 << 22) + 512
    assert int(out[0]) == int(a[0]) * int(b[0]) % cfg.p


def test_nearly_full_last_chunk_inverse(golden):
    """Vectors whose last chunk is nearly full (few columns c >= h) solve
    those columns one per CTA (k_col1_inv): the inverse against the oracle
    at 2^22 - j, and exact round trips of uniform batches and of longer
    vectors on all three word types (the forward is pinned elsewhere)."""
    cfg = T.default_config()
    for n in ((1 << 22) - 1, (1 << 22) - 37):
        z = gen(n + 5, cfg.p, n)
        assert np.array_equal(run(T.itft, z, cfg), O.itft(z, cfg.p, cfg.omegaK, cfg.K)), n
    cases = [("p998244353", (1 << 23) - 3, 1), ("p998244353", (3 << 21) - 2, 2), ("p998244353", (1 << 22) - 140, 2),
             ("p3221225473", (1 << 24) - 1, 1), ("p3221225473", (5 << 22) - 296, 1),
             ("p4179340454199820289", (1 << 22) - 1, 1), ("p4179340454199820289", (1 << 23) - 9, 2)]
    for key, n, count in cases:
        c = cfg_for(golden, key)
        flat = gen(n + count, c.p, n * count)
        d = device.to_words(flat, c)
        o = d.clone()
        device.tft_batch_(d, c, n=n, count=count)
        assert not torch.equal(d, o)
        device.tft_batch_(d, c, n=n, count=count, inverse=True)
        assert torch.equal(d, o), (key, n, count)
        plan = device.BatchPlan(c, [n] * count)
        plan.execute(d)
        plan.execute(d, inverse=True)
        assert torch.equal(d, o), (key, n, count, "plan")


def test_two_pass_products_with_zero_padded_operands(golden):
    """Two-pass products whose operands leave the column networks' top one
    or two layers with zero upper rows (k_colc_fwd ZT = 0, 1, 2 in every
    combination, operands much shorter and almost as long as the product),
    on both u32 word types and u64, against the oracle's product."""
    shapes = ((150000, 150001), (299990, 12), (5, 280000), (100000, 190000), (70000, 70000), (262144, 1))
    for key in ("p998244353", "p3221225473", "p4179340454199820289"):
        cfg = cfg_for(golden, key)
        for la, lb in shapes[:3] if key != "p998244353" else shapes:
            a = gen(la + 3, cfg.p, la)
            b = gen(lb + 7, cfg.p, lb)
            out = np.zeros(la + lb - 1, dtype=np.uint64)
            T.multiply(a, b, out, cfg)
            assert np.array_equal(out, O.multiply(a, b, cfg.p, cfg.omegaK, cfg.K)), (key, la, lb)


def test_extreme_residues_against_oracle(golden):
    """Inputs made of the extreme residues 0, 1, p - 1 and (p - 1) / 2 (all
    equal, alternating, and one hot) push the lazy and wide words of the
    rounds to the ends of their ranges -- for p = 3221225473 the carries of
    the 32-bit sums.  Tile, cluster and two-pass plans, forward and inverse,
    on the three word types, against the oracle."""
    for key in ("p998244353", "p3221225473", "p4179340454199820289"):
        cfg = cfg_for(golden, key)
        p = cfg.p
        for n in (999, 16385, 40000, 150001):
            pats = [np.full(n, p - 1, dtype=np.uint64),
                    np.where(np.arange(n) % 2 == 0, p - 1, 0).astype(np.uint64),
                    np.where(np.arange(n) % 3 == 0, (p - 1) // 2, p - 1).astype(np.uint64),
                    np.concatenate([np.zeros(n - 1, dtype=np.uint64), np.array([p - 1], dtype=np.uint64)]),
                    np.ones(n, dtype=np.uint64)]
            for i, x in enumerate(pats):
                y = run(T.tft, x, cfg)
                assert np.array_equal(y, O.tft(x, p, cfg.omegaK, cfg.K)), (key, n, i)
                assert np.array_equal(run(T.itft, x, cfg), O.itft(x, p, cfg.omegaK, cfg.K)), (key, n, i, "inv")
