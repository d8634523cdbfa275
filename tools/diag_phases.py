import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import backend
cfg = T.default_config()
lib = backend.load()
f = lib.tftb_debug_cluster_timing
f.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
for n in (49152, 65536):
    cnt = 4096
    G = (n + 16383) // 16384
    d = torch.randint(0, cfg.p, (cnt * n,), dtype=torch.int32, device="cuda")
    t = torch.zeros(cnt * G * 8, dtype=torch.int64, device="cuda")
    for _ in range(2):
        backend.check(f(cfg.p, cfg.omegaK, cfg.K, d.data_ptr(), n, cnt, t.data_ptr()))
    a = t.cpu().numpy().reshape(-1, 8).astype(np.float64)
    t0 = a[:, 0].min()
    dur = (a[:, 6].max() - t0) / 1e3
    ph = np.diff(a[:, :7], axis=1) / 1e3
    names = ["load", "sync1", "cross", "sync2", "rounds", "store"]
    print(f"n={n} G={G} kernel span {dur:.1f} us; per-CTA mean us: " + ", ".join(f"{nm} {ph[:, i].mean():.2f}" for i, nm in enumerate(names)),
          f"| CTA lifetime {np.mean(a[:, 6] - a[:, 0]) / 1e3:.2f} us, sum over CTAs / (444 slots) {np.sum(a[:, 6] - a[:, 0]) / 1e3 / 444:.1f} us")
