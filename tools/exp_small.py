"""Throughput of the one-CTA tile path: uniform batches of n = 2^t."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import device
cfg = T.default_config()
for n in [int(a) for a in sys.argv[1:]] or [1 << 14, 12288, 1 << 13]:
    cnt = (200 << 20) // n
    d = torch.randint(0, cfg.p, (cnt * n,), dtype=torch.int32, device="cuda")
    o = d.clone()
    for inv in (0, 1):
        for _ in range(3):
            device.tft_batch_(d, cfg, n=n, count=cnt, inverse=bool(inv))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 5
        ev[0].record()
        for _ in range(reps):
            device.tft_batch_(d, cfg, n=n, count=cnt, inverse=bool(inv))
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / reps
        bfly = cnt * n / 2 * (n.bit_length() - 1)
        print(f"n={n} inv={inv} cnt={cnt} {ms:.3f} ms  {cnt * n / ms / 1e6:.1f} Gcoeff/s  "
              f"{bfly / ms / 1e9 / 148 / 1.965e6 * 1e3:.2f} bfly/clk/SM  {8 * cnt * n / ms / 1e9:.0f} GB/s")
