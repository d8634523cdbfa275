"""Single and batched n = 2^k + r transforms vs 2^k (p2r overhead)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import device
for p, ks in ((998244353, (20, 22)), (469762049, (24,))):
    cfg = T.default_config() if p == 998244353 else T.config_for_modulus(p)
    for k in ks:
        for n in (1 << k, (1 << k) + 1, (1 << k) + 4):
            for batch in (1, max(1, (1 << 26) // n)):
                d = torch.randint(0, p, (batch * n,), dtype=torch.int32, device="cuda")
                plan = device.BatchPlan(cfg, np.full(batch, n))
                ts = []
                for inv in (False, True):
                    for _ in range(3):
                        plan.execute(d, inverse=inv)
                    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                    e[0].record()
                    for _ in range(10):
                        plan.execute(d, inverse=inv)
                    e[1].record()
                    torch.cuda.synchronize()
                    ts.append(e[0].elapsed_time(e[1]) / 10 * 1e3)
                print(f"p={p} n={n} batch={batch}: fwd {ts[0]:.1f} us inv {ts[1]:.1f} us ({batch * n / ts[0] / 1e3:.1f} / {batch * n / ts[1] / 1e3:.1f} Gcoeff/s)")
                del d, plan
