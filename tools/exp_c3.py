"""Config-3 single transforms (fwd + inv) for ncu / timing: python tools/exp_c3.py p n [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import device
p, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = T.config_for_modulus(p) if p != 998244353 else T.default_config()
d = torch.randint(0, 1 << 30, (n,), dtype=torch.int32, device="cuda")
d.remainder_(p if p < (1 << 31) else (1 << 30))
o = d.clone()
plan = device.BatchPlan(cfg, np.array([n]))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for r in range(reps):
    ev[0].record(); plan.execute(d); ev[1].record(); plan.execute(d, inverse=True); ev[2].record()
    torch.cuda.synchronize()
    print(f"p={p} n={n} fwd {ev[0].elapsed_time(ev[1])*1e3:.1f} us inv {ev[1].elapsed_time(ev[2])*1e3:.1f} us")
assert torch.equal(d, o)
