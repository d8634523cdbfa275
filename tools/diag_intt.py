import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import backend
cfg = T.default_config(); p = cfg.p
lib = backend.load()
f = lib.tftb_debug_intt_tile
f.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
for t in range(1, 15):
    R = 1 << t
    y = np.random.default_rng(t).integers(0, p, R, dtype=np.uint64)
    d = torch.from_numpy(y.astype(np.uint32).view(np.int32).copy()).cuda()
    backend.check(f(p, cfg.omegaK, cfg.K, d.data_ptr(), t))
    got = d.cpu().numpy().view(np.uint32).astype(np.uint64)
    x = y.copy(); T.itft(x, cfg)
    print("t", t, "bad", int((got != x).sum()), "ratio", [int(a) * pow(int(b), p - 2, p) % p for a, b in zip(got[:2], x[:2])])
