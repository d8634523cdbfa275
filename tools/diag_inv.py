import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1001_5272_b200 as T
from oracle import oracle as O
cfg = T.default_config()
for n in [131073, 150001, 262143, 262145, 300001, 524287, 524289, 600001, 1000001, 1048575, 1048577, 2000001]:
    z = np.random.default_rng(n).integers(0, cfg.p, n, dtype=np.uint64)
    a = z.copy(); T.itft(a, cfg)
    want = O.itft(z, cfg.p, cfg.omegaK, cfg.K)
    bad = np.nonzero(a != want)[0]
    l = (n - 1).bit_length(); l0 = min(l // 2, 9); l1 = l - l0
    C = 1 << l1; K = n >> l1; h = n & (C - 1)
    print(n, "l0", l0, "l1", l1, "K", K, "h", h, "bad", bad.size, (bad[:5], bad[:5] % C, bad[:5] // C) if bad.size else "")
