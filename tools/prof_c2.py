"""Small config-2 run for ncu (512 vectors, fwd + inv, 2 reps)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import device
cfg = T.default_config()
nvec = int(sys.argv[1]) if len(sys.argv) > 1 else 512
rng = np.random.default_rng(1)
lens = rng.integers(2**15 + 1, 2**16 + 1, nvec)
flat = rng.integers(0, cfg.p, int(lens.sum()), dtype=np.uint64)
d = device.to_words(flat, cfg)
o = d.clone()
for _ in range(2):
    device.tft_batch_(d, cfg, lengths=lens)
    device.tft_batch_(d, cfg, lengths=lens, inverse=True)
torch.cuda.synchronize()
assert torch.equal(d, o)
print("ok")
