import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1001_5272_b200 as T
from oracle import oracle as O
cfg = T.default_config()
for n in [131072, 131072 + 512, 131072 + 1024, 200000]:
    z = np.random.default_rng(n).integers(0, cfg.p, n, dtype=np.uint64)
    a = z.copy(); T.itft(a, cfg)
    w = O.itft(z, cfg.p, cfg.omegaK, cfg.K)
    bad = np.nonzero(a != w)[0]
    f = O.tft(z, cfg.p, cfg.omegaK, cfg.K); b = f.copy(); T.itft(b, cfg)
    print(os.environ.get("TFTB_FORCE_L1"), n, "inv bad", bad.size, bad[:3], bad[-3:] if bad.size else "", "roundtrip bad", int((b != z).sum()))
