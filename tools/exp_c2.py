import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import device
cfg = T.default_config()
def tm(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for n in [16385, 32768, 32769, 40000, 49152, 49153, 57344, 65536]:
    cnt = 4096
    d = torch.randint(0, cfg.p, (cnt * n,), dtype=torch.int32, device="cuda")
    plan = device.BatchPlan(cfg, np.full(cnt, n))
    f = tm(lambda: plan.execute(d)); i = tm(lambda: plan.execute(d, inverse=True))
    print(f"n={n:6d} G={(n + 16383) // 16384} h={n % 16384:5d} fwd {f:.3f} ms ({cnt*n/f/1e6:.0f} Gc/s)  inv {i:.3f} ms ({cnt*n/i/1e6:.0f} Gc/s)")
    del d, plan
