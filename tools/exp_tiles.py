"""Uniform batches (~2^28 words) of small lengths: tile-path fwd/inv Gcoeff/s."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import device
cfg = T.default_config()
for n in [int(a) for a in sys.argv[1:]] or [1027, 1252, 2267, 4107, 9067, 13472]:
    batch = (1 << 28) // n
    d = torch.randint(0, cfg.p, (batch * n,), dtype=torch.int32, device="cuda")
    plan = device.BatchPlan(cfg, np.full(batch, n))
    ts = []
    for inv in (False, True):
        for _ in range(2):
            plan.execute(d, inverse=inv)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        for _ in range(3):
            plan.execute(d, inverse=inv)
        e[1].record()
        torch.cuda.synchronize()
        ts.append(e[0].elapsed_time(e[1]) / 3)
    print(f"n={n}: fwd {batch * n / ts[0] / 1e6:.0f} inv {batch * n / ts[1] / 1e6:.0f} Gcoeff/s")
    del d, plan
