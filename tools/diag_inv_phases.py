"""Phase timestamps of the fused cluster-range inverse (k_cli_chunks):
    python tools/diag_inv_phases.py [n ...]"""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1001_5272_b200 as T  # noqa: E402
from paper_1001_5272_b200 import backend  # noqa: E402
cfg = T.default_config()
lib = backend.load()
f = lib.tftb_debug_cluster_timing
f.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
              ctypes.c_void_p, ctypes.c_int]
for n in [int(x) for x in sys.argv[1:]] or (40000, 49152, 57344, 65530):
    cnt = 4096
    G = (n + 16383) // 16384
    d = torch.randint(0, cfg.p, (cnt * n,), dtype=torch.int32, device="cuda")
    t = torch.zeros(cnt * G * 8, dtype=torch.int64, device="cuda")
    for _ in range(2):
        t.zero_()
        backend.check(f(cfg.p, cfg.omegaK, cfg.K, d.data_ptr(), n, cnt, t.data_ptr(), 1))
    a = t.cpu().numpy().reshape(cnt * G, 8).astype(np.float64)
    span = (a[:, 3].max() - a[:, 0].min()) / 1e3
    last = a[a[:, 7] > 0]
    q = lambda arr, i, j: np.mean(arr[:, j] - arr[:, i]) / 1e3
    print(f"inv n={n} G={G}: chunk CTA load {q(a, 0, 1):.2f}, rounds {q(a, 1, 2):.2f}, store+ticket {q(a, 2, 3):.2f} us; "
          f"last CTA ({len(last)}): cols>=h {q(last, 3, 4):.2f}, load {q(last, 4, 5):.2f}, phases23 {q(last, 5, 6):.2f}, "
          f"cols<h {q(last, 6, 7):.2f} us; span {(np.max(a[:, 7]) - a[:, 0].min()) / 1e3:.0f} us")
