"""A batched transform at one length (fwd + inv), for ncu launch lists:
    python tools/prof_size.py n [count] [p]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1001_5272_b200 as T  # noqa: E402
import workloads as W  # noqa: E402
from paper_1001_5272_b200 import device  # noqa: E402
n = int(sys.argv[1])
cnt = int(sys.argv[2]) if len(sys.argv) > 2 else max(1, (1 << 28) // n)
p = int(sys.argv[3]) if len(sys.argv) > 3 else W.P_DEFAULT
cfg = T.default_config() if p == W.P_DEFAULT else T.config_for_modulus(p)
d = device.to_words(W.words(4, p, n * cnt), cfg)
o = d.clone()
plan = device.BatchPlan(cfg, np.full(cnt, n))
for _ in range(2):
    plan.execute(d)
    plan.execute(d, inverse=True)
torch.cuda.synchronize()
assert torch.equal(d, o)
print("ok")
