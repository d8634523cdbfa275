"""Compare the large-path inverse's intermediate states with a numpy model."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1001_5272_b200 as T
from oracle import oracle as O
cfg = T.default_config(); p = cfg.p
l1 = int(os.environ["TFTB_FORCE_L1"]); C = 1 << l1
stop = int(os.environ.get("TFTB_DEBUG_STOP", "9"))
n = int(sys.argv[1])
Y = np.random.default_rng(n).integers(0, p, n, dtype=np.uint64)
xt = O.itft(Y, p, cfg.omegaK, cfg.K)            # true coefficients
K, h = n >> l1, n & (C - 1)
R = 1 << ((n - 1).bit_length() - l1)
# z[c + k C] = sum_i xt[c + i C] omega_k^i  (column transforms), rows k <= K
om = np.array([O.omega(k, p, cfg.omegaK, cfg.K) for k in range(K + 1)], dtype=object)
z = np.zeros((K + 1) * C, dtype=object)
for c in range(C):
    col = [int(v) for v in xt[c::C]]
    for k in range(K + 1):
        acc = 0
        for i in reversed(range(len(col))):
            acc = (acc * int(om[k]) + col[i]) % p
        z[c + k * C] = acc
a = Y.copy(); T.itft(a, cfg)
a = a.astype(object)
if stop == 1:
    bad = [i for i in range(K * C) if a[i] != z[i]]
    print("step1 chunks<K bad", len(bad), bad[:5])
elif stop == 2:
    bad = [i for i in range(K * C) if i % C >= h and a[i] != xt[i]]
    print("step2 cols>=h x bad", len(bad), bad[:5], sorted(set(i % C for i in bad))[:10])
elif stop == 3:
    bad = [c for c in range(h) if a[K * C + c] != z[K * C + c]]
    print("step3 last chunk head bad", len(bad), bad[:10])
else:
    bad = np.nonzero(a != xt.astype(object))[0]
    print("final bad", len(bad))
