"""Batched transforms at one length per size class, for ncu pipe tables:
    python tools/prof_tiles.py [T ...]     (default T = 10..17)
n = 2^T - 3 (never a power of two), ~2^24 words per launch, fwd then inv."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1001_5272_b200 as T  # noqa: E402
import workloads as W  # noqa: E402
from paper_1001_5272_b200 import device  # noqa: E402
cfg = T.default_config()
for t in [int(a) for a in sys.argv[1:]] or range(10, 18):
    n = (1 << t) - 3
    cnt = max(1, (1 << 24) // n)
    x = W.words(4, cfg.p, n * cnt)
    d = device.to_words(x, cfg)
    o = d.clone()
    plan = device.BatchPlan(cfg, np.full(cnt, n))
    plan.execute(d)
    plan.execute(d, inverse=True)
    torch.cuda.synchronize()
    assert torch.equal(d, o), t
print("ok")
