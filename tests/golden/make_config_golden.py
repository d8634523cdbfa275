"""Generate tests/golden/configs.json: sha256 digests of the REFERENCE's own
outputs on every BASELINE config's pinned inputs.

Run in the build container (where /root/reference exists):

    make -C oracle ref
    python tests/golden/make_config_golden.py      # ~10 min on 8 cores

The transforms are the reference's compiled Cython kernels
(`_kernels.pyx:415-430` tft/itft, `:433-480` multiply, built from the
reference source by oracle/Makefile into oracle/_ref/).  They release the GIL,
so independent vectors run on a thread pool.  Inputs come from
`workloads.py` (the generator BASELINE.md §3 pins), so the GPU box can
regenerate them; only the digests travel (tests/test_gpu_configs.py).

Digest = sha256 of the output words as little-endian uint64.
  config 2: the whole seed-1 batch (4096 vectors, 201,947,138 words) after a
            per-vector tft, and after a per-vector itft of the same input words.
  config 3: tft and itft of the seed-2 vector at each of the five lengths at
            p = 3221225473, and the five default-prime lengths.
  config 4: multiply of pairs 0, 1 and 255 of the seed-3 stream.
  config 5: all 64 lengths on both legs; vector 0 of each launch (and
            vector 1 where 2n <= 2^25), tft and itft of the input words.
"""

import hashlib
import json
import os
import sys
import time
from array import array
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import workloads as W  # noqa: E402
from oracle.oracle import ref_kernels  # noqa: E402

K_ = ref_kernels()
assert K_ is not None, "build the reference kernels first: make -C oracle ref"

sys.path.insert(0, "/root/reference/pkg/src")
import tftmul  # noqa: E402  (only for config_for_modulus: the reference's own ring discovery)


def ring(p):
    if p == W.P_DEFAULT:
        c = tftmul.default_config()
    else:
        c = tftmul.config_for_modulus(p)
    return c.p, c.omegaK, c.K


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def ref_inplace(buf, off, n, p, top, K, inverse):
    mv = memoryview(buf)
    if inverse:
        K_.itft(mv, off, n, p, top, K, (p + 1) >> 1)
    else:
        K_.tft(mv, off, n, p, top, K)


def ref_vec(x, p, inverse):
    p, top, K = ring(p)
    buf = array("Q", np.ascontiguousarray(x, dtype=np.uint64).tobytes())
    ref_inplace(buf, 0, len(buf), p, top, K, inverse)
    return np.frombuffer(buf, dtype=np.uint64)


def main():
    t0 = time.time()
    cores = os.cpu_count() or 1
    out = {"generator": "workloads.py (numpy default_rng(seed).integers(0, p, n, dtype=uint64))",
           "digest": "sha256 of output words, little-endian uint64",
           "source": "reference compiled kernels (_kernels.pyx via oracle/_ref)",
           "rings": {}, "config2": {}, "config3": [], "config4": [], "config5": []}
    for p in (W.P_DEFAULT, W.P_C3, W.P_U64):
        out["rings"][str(p)] = list(ring(p))

    def log(msg):
        print(f"[{time.time() - t0:7.1f}s] {msg}", flush=True)

    # ---- config 5 and config 3 tasks, largest first on the pool
    tasks = []
    for n in W.c5_lengths():
        for leg in ("u32", "u64"):
            cnt = 2 if 2 * n <= (1 << 25) else 1
            tasks.append(("c5", n, leg, cnt))
    for n in W.C3_LENGTHS:
        tasks.append(("c3", n, W.P_C3, 1))
    for n in W.C3_DEFAULT_LENGTHS:
        tasks.append(("c3", n, W.P_DEFAULT, 1))
    tasks.sort(key=lambda t: -t[1] * t[3])

    def run_task(t):
        kind, n, arg, cnt = t
        if kind == "c5":
            p = W.c5_prime(n, arg)
            x = W.c5(n, arg, cnt)
        else:
            p = arg
            x = W.c3(n, p)
        rec = {"n": n, "p": p}
        if kind == "c5":
            rec.update({"leg": arg, "vectors": cnt, "batch": W.c5_batch(n, 4 if arg == "u32" else 8)})
        fw, iv = [], []
        for v in range(cnt):
            xv = x[v * n:(v + 1) * n]
            f = ref_vec(xv, p, False)
            fw.append(sha(f))
            if v == 0:
                rec["tft_head"] = [int(a) for a in f[:4]]
            iv.append(sha(ref_vec(xv, p, True)))
        rec["tft"] = fw
        rec["itft"] = iv
        log(f"{kind} n={n} {arg} x{cnt}")
        return kind, rec

    with ThreadPoolExecutor(cores) as ex:
        for kind, rec in ex.map(run_task, tasks):
            (out["config5"] if kind == "c5" else out["config3"]).append(rec)
    out["config5"].sort(key=lambda r: (r["leg"], r["n"]))
    out["config3"].sort(key=lambda r: (r["p"], r["n"]))

    # ---- config 2: the whole batch, per-vector transforms on the pool
    lens, flat = W.c2(1)
    offs = np.concatenate(([0], np.cumsum(lens)[:-1]))
    p, top, K = ring(W.P_DEFAULT)
    rec = {"vectors": int(lens.size), "words": int(lens.sum())}
    for name, inv in (("tft", False), ("itft", True)):
        buf = array("Q", flat.tobytes())

        def one(i, buf=buf, inv=inv):
            ref_inplace(buf, int(offs[i]), int(lens[i]), p, top, K, inv)
        with ThreadPoolExecutor(cores) as ex:
            list(ex.map(one, range(lens.size)))
        res = np.frombuffer(buf, dtype=np.uint64)
        rec[name] = sha(res)
        rec[name + "_head"] = [int(a) for a in res[:4]]
        rec[name + "_last_vector"] = sha(res[int(offs[-1]):])
        log(f"config 2 {name}")
    out["config2"] = rec

    # ---- config 4: pairs 0, 1, 255
    pairs = list(W.c4_pairs([0, 1, 255]))

    def mul(item):
        k, a, b = item
        A, B = array("Q", a.tobytes()), array("Q", b.tobytes())
        X = array("Q", bytes(8 * (len(A) + len(B) - 1)))
        K_.multiply(memoryview(A), memoryview(B), memoryview(X), p, top, K, (p + 1) >> 1)
        x = np.frombuffer(X, dtype=np.uint64)
        log(f"config 4 pair {k}")
        return {"pair": k, "la": len(A), "lb": len(B), "x": sha(x), "x_head": [int(v) for v in x[:4]]}
    with ThreadPoolExecutor(3) as ex:
        out["config4"] = list(ex.map(mul, pairs))

    with open(os.path.join(HERE, "configs.json"), "w") as f:
        json.dump(out, f, indent=0, separators=(",", ":"))
    log("wrote configs.json")


if __name__ == "__main__":
    main()
