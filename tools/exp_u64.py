"""u64 leg timing at a few config-5 sizes: python tools/exp_u64.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1001_5272_b200 as T
import workloads as W
from paper_1001_5272_b200 import device
p = 4179340454199820289
cfg = T.config_for_modulus(p)
def ev_time(fn, reps=5):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]
for n, batch in [(7438, 4000), (29742, 1000), (65664, 500), (118930, 300), (475566, 80), (1901646, 20), (7604114, 6), (30406570, 2)]:
    d = device.to_words(W.c3(n, p), cfg).repeat(batch)
    o = d.clone()
    plan = device.BatchPlan(cfg, [n] * batch)
    plan.execute(d); plan.execute(d, inverse=True)
    assert torch.equal(d, o)
    tf = ev_time(lambda: plan.execute(d)); ti = ev_time(lambda: plan.execute(d, inverse=True))
    print(f"  u64 n={n} x{batch}: fwd {n*batch/tf/1e6:.1f} inv {n*batch/ti/1e6:.1f} Gcoeff/s")
