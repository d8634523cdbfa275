"""Bit-exact parity on every BASELINE config at full size: the CUDA path
against sha256 digests of the REFERENCE's own outputs on the same pinned
inputs (tests/golden/configs.json, made by make_config_golden.py from the
reference's compiled kernels, `_kernels.pyx:415-480`).

  config 2: the whole seed-1 batch (4096 vectors, 201,947,138 words), tft
            and itft of the input words (through a BatchPlan, the bench path)
  config 3: the five lengths 2^24 .. 2^25+1 at p = 3221225473 and the five
            default-prime lengths 2^22 .. 2^23, tft and itft (seed 2)
  config 4: products of pairs 0, 1 and 255 of the seed-3 stream (pair 0
            through the reference-facing multiply(), 1 and 255 on device)
  config 5: all 64 lengths on both legs (u32 and the 62-bit prime), the
            head vectors of each launch, tft and itft (seed 4)
"""

import json
import os

import numpy as np
import pytest

from conftest import sha

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_1001_5272_b200 as T  # noqa: E402
import workloads as W  # noqa: E402
from paper_1001_5272_b200 import device  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def cg():
    with open(os.path.join(HERE, "golden", "configs.json")) as f:
        return json.load(f)


def ring(cg, p):
    pp, top, K = cg["rings"][str(p)]
    return T.RingConfig(pp, top, K)


def vec_digests(d, cfg, n, cnt):
    got = device.from_words(d, cfg)
    return [sha(got[v * n:(v + 1) * n]) for v in range(cnt)]


def test_config2_full_batch(cg):
    rec = cg["config2"]
    cfg = ring(cg, W.P_DEFAULT)
    lens, flat = W.c2(1)
    assert int(lens.sum()) == rec["words"]
    plan = device.BatchPlan(cfg, lens)
    d = device.to_words(flat, cfg)
    plan.execute(d)
    out = device.from_words(d, cfg)
    assert [int(v) for v in out[:4]] == rec["tft_head"]
    assert sha(out) == rec["tft"]
    plan.execute(d, inverse=True)
    assert torch.equal(d, device.to_words(flat, cfg))
    plan.execute(d, inverse=True)  # itft of the input words themselves
    assert sha(device.from_words(d, cfg)) == rec["itft"]


@pytest.mark.parametrize("which", ["p3221225473", "p998244353"])
def test_config3_lengths(cg, which):
    recs = [r for r in cg["config3"] if f"p{r['p']}" == which]
    assert len(recs) == 5
    for rec in recs:
        n, cfg = rec["n"], ring(cg, rec["p"])
        x = W.c3(n, rec["p"])
        d = device.to_words(x, cfg)
        device.tft_batch_(d, cfg, n=n)
        assert vec_digests(d, cfg, n, 1) == rec["tft"], ("tft", n)
        device.tft_batch_(d, cfg, n=n, inverse=True)
        assert torch.equal(d, device.to_words(x, cfg)), ("round trip", n)
        device.tft_batch_(d, cfg, n=n, inverse=True)
        assert vec_digests(d, cfg, n, 1) == rec["itft"], ("itft", n)


def test_config4_pairs(cg):
    cfg = T.default_config()
    want = {r["pair"]: r for r in cg["config4"]}
    for k, a, b in W.c4_pairs(sorted(want)):
        rec = want[k]
        if k == 0:  # through the reference-facing API (host uint64 buffers)
            x = np.zeros(a.size + b.size - 1, dtype=np.uint64)
            T.multiply(a, b, x, cfg)
        else:
            dx = torch.zeros(a.size + b.size - 1, dtype=device.word_dtype(cfg), device="cuda")
            device.multiply_batch(device.to_words(a, cfg), device.to_words(b, cfg), dx, cfg, 1, a.size, b.size)
            x = device.from_words(dx, cfg)
        assert [int(v) for v in x[:4]] == rec["x_head"], k
        assert sha(x) == rec["x"], k


@pytest.mark.parametrize("leg", ["u32", "u64"])
def test_config5_sweep(cg, leg):
    recs = [r for r in cg["config5"] if r["leg"] == leg]
    assert len(recs) == 64
    for rec in recs:
        n, cnt, cfg = rec["n"], rec["vectors"], ring(cg, rec["p"])
        x = W.c5(n, leg, cnt)
        d = device.to_words(x, cfg)
        device.tft_batch_(d, cfg, n=n, count=cnt)
        assert vec_digests(d, cfg, n, cnt) == rec["tft"], ("tft", leg, n)
        d = device.to_words(x, cfg)
        device.tft_batch_(d, cfg, n=n, count=cnt, inverse=True)
        assert vec_digests(d, cfg, n, cnt) == rec["itft"], ("itft", leg, n)
        del d
