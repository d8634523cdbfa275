"""Batched fwd/inv Gcoeff/s at given lengths (pinned inputs, ~2^25 words per
launch unless a count is given): python tools/time_sizes.py [p] n1 n2 ...
(TFTB_LIB selects a library build, for A/B runs)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1001_5272_b200 as T  # noqa: E402
import workloads as W  # noqa: E402
from paper_1001_5272_b200 import device  # noqa: E402

args = [int(a) for a in sys.argv[1:]]
p = W.P_DEFAULT
if args and args[0] in (W.P_C3, W.P_U64, W.P_DEFAULT, 469762049):
    p = args.pop(0)
cfg = T.default_config() if p == W.P_DEFAULT else T.config_for_modulus(p)
for n in args:
    cnt = max(1, (1 << 25) // n)
    d = device.to_words(W.words(4, p, n * cnt), cfg)
    plan = device.BatchPlan(cfg, np.full(cnt, n))
    for _ in range(2):
        plan.execute(d)
        plan.execute(d, inverse=True)
    torch.cuda.synchronize()
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record()
    for _ in range(5):
        plan.execute(d)
    b.record()
    for _ in range(5):
        plan.execute(d, inverse=True)
    c.record()
    torch.cuda.synchronize()
    print(p, n, cnt, "fwd", round(cnt * n * 5 / a.elapsed_time(b) / 1e6, 1), "inv", round(cnt * n * 5 / b.elapsed_time(c) / 1e6, 1),
          flush=True)
