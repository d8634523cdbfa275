"""Small config-4 run for ncu: `pairs` products 2,500,001 x 1,750,004."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import device
cfg = T.default_config()
pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 16
la, lb = 2500001, 1750004
r = la + lb - 1
a = torch.randint(0, cfg.p, (pairs * la,), dtype=torch.int32, device="cuda")
b = torch.randint(0, cfg.p, (pairs * lb,), dtype=torch.int32, device="cuda")
x = torch.empty(pairs * r, dtype=torch.int32, device="cuda")
y = torch.empty(pairs * r, dtype=torch.int32, device="cuda")
for _ in range(2):
    device.multiply_batch(a, b, x, cfg, pairs, la, lb, scratch=y)
torch.cuda.synchronize()
print("ok")
