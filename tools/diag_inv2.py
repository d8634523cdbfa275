import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1001_5272_b200 as T
from oracle import oracle as O
cfg = T.default_config()
for n in [131073, 262145, 600001]:
    z = np.random.default_rng(n).integers(0, cfg.p, n, dtype=np.uint64)
    a = z.copy(); T.itft(a, cfg)
    f = z.copy(); T.tft(f, cfg)
    print(os.environ.get("TFTB_FORCE_L1"), n, "inv bad", int((a != O.itft(z, cfg.p, cfg.omegaK, cfg.K)).sum()),
          "fwd bad", int((f != O.tft(z, cfg.p, cfg.omegaK, cfg.K)).sum()))
