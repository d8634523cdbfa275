"""One large transform (fwd + inv) for ncu: python tools/prof_c3.py [n] [p]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1001_5272_b200 as T  # noqa: E402
import workloads as W  # noqa: E402
from paper_1001_5272_b200 import device  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
p = int(sys.argv[2]) if len(sys.argv) > 2 else W.P_C3
cfg = T.config_for_modulus(p) if p != W.P_DEFAULT else T.default_config()
x = W.c3(n, p)
d = device.to_words(x, cfg)
o = d.clone()
plan = device.BatchPlan(cfg, [n])
for _ in range(2):
    plan.execute(d)
    plan.execute(d, inverse=True)
torch.cuda.synchronize()
assert torch.equal(d, o)
print("ok")
