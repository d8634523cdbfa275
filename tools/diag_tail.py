"""Phase stamps of the single-CTA tail of a large inverse (k_col1_inv, k_last_inv):
    python tools/diag_tail.py [p n ...]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import backend, device
import workloads as W
lib = backend.load()
lib.tftb_debug_tail_timing.argtypes = [ctypes.c_void_p]
args = [int(x) for x in sys.argv[1:]] or [W.P_C3, (1 << 25) - 1, 998244353, (1 << 23) - 1]
for p, n in zip(args[::2], args[1::2]):
    cfg = T.config_for_modulus(p) if p != 998244353 else T.default_config()
    d = device.to_words(W.c3(n, p), cfg)
    plan = device.BatchPlan(cfg, [n])
    t = torch.zeros(16, dtype=torch.int64, device="cuda")
    lib.tftb_debug_tail_timing(t.data_ptr())
    for _ in range(3):
        plan.execute(d)
        plan.execute(d, inverse=True)
    torch.cuda.synchronize()
    lib.tftb_debug_tail_timing(None)
    a = t.cpu().numpy().astype(float) / 1e3
    print(f"p={p} n={n}: col1 load {a[1]-a[0]:.1f} rounds {a[2]-a[1]:.1f} phases23 {a[3]-a[2]:.1f} store {a[4]-a[3]:.1f} "
          f"colsum {a[5]-a[4]:.1f} | gap {a[8]-a[5]:.1f} | last load {a[9]-a[8]:.1f} phases23 {a[10]-a[9]:.1f} store {a[11]-a[10]:.1f} us")
