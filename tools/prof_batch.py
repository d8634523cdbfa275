"""A uniform two-pass batch (fwd + inv) for ncu: python tools/prof_batch.py p n count"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1001_5272_b200 as T
import workloads as W
from paper_1001_5272_b200 import device
p, n, count = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cfg = T.config_for_modulus(p) if p != W.P_DEFAULT else T.default_config()
d = device.to_words(W.c3(n, p), cfg).repeat(count)
o = d.clone()
plan = device.BatchPlan(cfg, [n] * count)
for _ in range(2):
    plan.execute(d)
    plan.execute(d, inverse=True)
torch.cuda.synchronize()
assert torch.equal(d, o)
print("ok")
