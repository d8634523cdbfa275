import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1001_5272_b200 as T
from oracle import oracle as O
cfg = T.default_config()
l1 = int(os.environ["TFTB_FORCE_L1"]); C = 1 << l1
for n in [131584, 200000]:
    z = np.random.default_rng(n).integers(0, cfg.p, n, dtype=np.uint64)
    a = z.copy(); T.itft(a, cfg)
    w = O.itft(z, cfg.p, cfg.omegaK, cfg.K)
    bad = np.nonzero(a != w)[0]
    K, h = n >> l1, n & (C - 1)
    cols = np.unique(bad % C); rows = np.unique(bad // C)
    print(l1, n, "K", K, "h", h, "bad cols", cols.size, cols[:8], cols[-4:], "rows", rows.size, rows[:5], rows[-3:])
