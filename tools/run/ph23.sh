python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t12.log 2>&1; tail -1 gpurun_out/t12.log
python tools/prof_tiles.py > /dev/null 2>&1
for lib in tools/variants/libtftb200_before.so paper_1001_5272_b200/libtftb200.so; do
  echo "== $lib" >> gpurun_out/ph23.txt
  TFTB_LIB=$lib python - >> gpurun_out/ph23.txt 2>&1 <<'PY'
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1001_5272_b200 as T, workloads as W
from paper_1001_5272_b200 import device
cfg = T.default_config()
for n in (1027, 2267, 4093, 8191, 13472, 16381, 40000, 57344, 65530):
    cnt = max(1, (1 << 25) // n)
    d = device.to_words(W.words(4, cfg.p, n * cnt), cfg)
    plan = device.BatchPlan(cfg, np.full(cnt, n))
    for _ in range(2): plan.execute(d); plan.execute(d, inverse=True)
    torch.cuda.synchronize()
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record()
    for _ in range(5): plan.execute(d)
    b.record()
    for _ in range(5): plan.execute(d, inverse=True)
    c.record(); torch.cuda.synchronize()
    print(n, 'fwd', round(cnt * n * 5 / a.elapsed_time(b) / 1e6, 1), 'inv', round(cnt * n * 5 / b.elapsed_time(c) / 1e6, 1))
PY
done
