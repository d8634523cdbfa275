import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import backend
cfg = T.default_config(); p = cfg.p
lib = backend.load()
f = lib.tftb_debug_itft_tile
f.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_uint32]
for t, wlog, h in [(7, 4, 68), (7, 0, 68), (8, 4, 136), (7, 4, 100), (7, 3, 68), (7, 1, 68), (9, 4, 256), (9, 4, 300)]:
    W = 1 << wlog; R = 1 << t
    rng = np.random.default_rng(t * 100 + h)
    tile = rng.integers(0, p, (R, W), dtype=np.uint64)
    tile[h:, :] = 0
    d = torch.from_numpy(tile.astype(np.uint32).view(np.int32).reshape(-1).copy()).cuda()
    backend.check(f(p, cfg.omegaK, cfg.K, d.data_ptr(), t, wlog, h))
    got = d.cpu().numpy().view(np.uint32).reshape(R, W)
    bad = 0
    for c in range(W):
        col = tile[:, c].copy()
        d1 = torch.from_numpy(col.astype(np.uint32).view(np.int32).copy()).cuda()
        backend.check(f(p, cfg.omegaK, cfg.K, d1.data_ptr(), t, 0, h))
        one = d1.cpu().numpy().view(np.uint32)
        x = col[:h].copy(); T.itft(x, cfg)  # reference via the full API
        bad += int((got[:h, c] != x).sum()) * 1000 + int((one[:h] != x).sum())
    print("t", t, "wlog", wlog, "h", h, "bad(interleaved*1000 + single)", bad)
