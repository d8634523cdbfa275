"""Twiddle-table size A/B (TFTB_ZB): config-4-shaped products, a config-5-shaped
two-pass batch and config-3 single transforms.  python tools/exp_zb.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import device
import workloads as W

def ev_time(fn, reps=5):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]

cfg = T.default_config()
pairs, la, lb = 64, 2500001, 1750004
r = la + lb - 1
a = torch.randint(0, cfg.p, (pairs * la,), dtype=torch.int32, device="cuda")
b = torch.randint(0, cfg.p, (pairs * lb,), dtype=torch.int32, device="cuda")
x = torch.empty(pairs * r, dtype=torch.int32, device="cuda")
y = torch.empty(pairs * r, dtype=torch.int32, device="cuda")
device.multiply_batch(a, b, x, cfg, pairs, la, lb, scratch=y)
t = ev_time(lambda: device.multiply_batch(a, b, x, cfg, pairs, la, lb, scratch=y))
print(f"zb={os.environ.get('TFTB_ZB')} config4 x{pairs}: {t:.2f} ms = {pairs / t * 1e3:.0f} products/s")
del a, b, x, y
for p, n, batch in [(998244353, 1901646, 141), (998244353, 7604114, 35), (998244353, 1 << 23, 1), (W.P_C3, 1 << 24, 1), (W.P_C3, (1 << 25) - 1, 1)]:
    c = T.config_for_modulus(p) if p != 998244353 else cfg
    d = device.to_words(W.c3(n, p), c).repeat(batch)
    plan = device.BatchPlan(c, [n] * batch)
    plan.execute(d); plan.execute(d, inverse=True)
    tf = ev_time(lambda: plan.execute(d)); ti = ev_time(lambda: plan.execute(d, inverse=True))
    print(f"  p={p} n={n} x{batch}: fwd {tf*1e3:.1f} us inv {ti*1e3:.1f} us  ({n*batch/tf/1e6:.1f} / {n*batch/ti/1e6:.1f} Gcoeff/s)")
