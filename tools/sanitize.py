"""Small runs of the round-2 paths (a quick exercise script; written for
compute-sanitizer, which is closed on this GPU pool, so it only checks the
round trips):
    python tools/sanitize.py
F32 wide rounds, step 2 by column (n = 2^k - j), whole-chunk inverses, and a
two-pass product whose operands are zero-padded (ZT column kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1001_5272_b200 as T
import workloads as W
from paper_1001_5272_b200 import device

for p in (W.P_DEFAULT, W.P_C3, 4179340454199820289):
    cfg = T.config_for_modulus(p) if p != W.P_DEFAULT else T.default_config()
    for n, count in (((1 << 22) - 1, 1), ((1 << 22) - 5, 2), (1 << 22, 1), (3 << 20, 1), ((1 << 22) + 1, 1), (70000, 3), (1000, 5)):
        flat = W.c3(n * count, p)
        d = device.to_words(flat, cfg)
        o = d.clone()
        device.tft_batch_(d, cfg, n=n, count=count)
        device.tft_batch_(d, cfg, n=n, count=count, inverse=True)
        assert torch.equal(d, o), (p, n, count)
    la, lb, pairs = 300001, 120004, 2
    r = la + lb - 1
    a = device.to_words(W.c3(pairs * la, p), cfg)
    b = device.to_words(W.c3(pairs * lb, p)[::-1].copy(), cfg)
    x = torch.empty(pairs * r, dtype=a.dtype, device="cuda")
    device.multiply_batch(a, b, x, cfg, pairs, la, lb)
    torch.cuda.synchronize()
    print("ok", p)
