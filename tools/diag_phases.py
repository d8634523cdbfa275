import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1001_5272_b200 as T
from paper_1001_5272_b200 import backend
cfg = T.default_config()
lib = backend.load()
f = lib.tftb_debug_cluster_timing
f.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]
names = {0: ["load", "sync1", "cross", "sync2", "rounds", "store", "-"],
         2: ["cone load", "sync", "-", "-", "rounds", "store", "-"],
         1: ["load", "intt", "sync1", "col1+publish", "exit sync", "phases23", "col2"]}
for inv in [2]:  # forward only (the split inverse has no phase stamps)
    for n in [int(x) for x in sys.argv[1:]] or (40000, 49152, 57344, 65536):
        cnt = 4096
        G = (n + 16383) // 16384
        d = torch.randint(0, cfg.p, (cnt * n,), dtype=torch.int32, device="cuda")
        t = torch.zeros(cnt * G * 8, dtype=torch.int64, device="cuda")
        for _ in range(2):
            backend.check(f(cfg.p, cfg.omegaK, cfg.K, d.data_ptr(), n, cnt, t.data_ptr(), 0 if inv == 2 else inv))
        a = t.cpu().numpy().reshape(-1, 8).astype(np.float64)
        last = 7 if inv == 1 else 6
        if inv == 1 and n % 16384 == 0:
            last = 4  # complete last chunk: the kernel ends after the first column solve
        if inv == 1 and n % 16384:
            # only the last CTA of a vector runs past the exit barrier
            b = a.reshape(cnt, G, 8)
            for role, sl, e in (("last CTA", b[:, G - 1], 7), ("others", b[:, :G - 1].reshape(-1, 8), 4)):
                q = np.diff(sl[:, :e + 1], axis=1) / 1e3
                print(f"    {role:9s}: life {np.mean(sl[:, e] - sl[:, 0]) / 1e3:.2f} us: "
                      + ", ".join(f"{nm} {q[:, i].mean():.2f}" for i, nm in enumerate(names[inv][:e])))
            continue
        if inv == 2:
            d_ = lambda i, j: np.mean(a[:, j] - a[:, i]) / 1e3
            print(f"fwd(no-cluster) n={n} G={G} span {(a[:, 6].max() - a[:, 0].min()) / 1e3:.0f} us; CTA life "
                  f"{d_(0, 6):.2f} us: cone load {d_(0, 1):.2f}, sync {d_(1, 2):.2f}, rounds {d_(2, 5):.2f}, "
                  f"store {d_(5, 6):.2f}")
            continue
        ph = np.diff(a[:, :last + 1], axis=1) / 1e3
        print(f"inv={inv} n={n} G={G} span {(a[:, last].max() - a[:, 0].min()) / 1e3:.0f} us; CTA life {np.mean(a[:, last] - a[:, 0]) / 1e3:.2f} us: "
              + ", ".join(f"{nm} {ph[:, i].mean():.2f}" for i, nm in enumerate(names[inv][:last])))
        del d, t
