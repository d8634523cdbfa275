"""One large transform (fwd + inv) for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import device
cfg = T.default_config()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8388607
x = np.random.default_rng(2).integers(0, cfg.p, n, dtype=np.uint64)
d = device.to_words(x, cfg); o = d.clone()
plan = device.BatchPlan(cfg, [n])
for _ in range(2):
    plan.execute(d); plan.execute(d, inverse=True)
torch.cuda.synchronize()
assert torch.equal(d, o)
print("ok")
