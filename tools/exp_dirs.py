"""Config-2 batch: forward and inverse passes, a few times each (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import device
cfg = T.default_config()
rng = np.random.default_rng(1)
lens = rng.integers(2**15 + 1, 2**16 + 1, 4096)
flat = rng.integers(0, cfg.p, int(lens.sum()), dtype=np.uint64)
d = device.to_words(flat, cfg)
plan = device.BatchPlan(cfg, lens)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    plan.execute(d)
    plan.execute(d, inverse=True)
torch.cuda.synchronize()
print("total coeffs", int(lens.sum()), "G3", int((lens <= 49152).sum()), "G4", int((lens > 49152).sum()))
