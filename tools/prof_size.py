"""One uniform batch (~2^28 words) of length n, fwd + inv twice (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import device
cfg = T.default_config()
n = int(sys.argv[1])
batch = (1 << 28) // n
d = torch.randint(0, cfg.p, (batch * n,), dtype=torch.int32, device="cuda")
plan = device.BatchPlan(cfg, np.full(batch, n))
for _ in range(2):
    plan.execute(d)
    plan.execute(d, inverse=True)
torch.cuda.synchronize()
print("ok")
