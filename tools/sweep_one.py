import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import torch
from paper_2303_02317_b200 import _native
T = 4096; n = 1
cap = int(sys.argv[1]) if len(sys.argv) > 1 else T + 2
db = _native.DeviceBatch(np.full(n, 2, np.int8), np.full(n, 100.0), np.full(n, 100.0), np.full(n, 0.05), np.zeros(n), np.full(n, 0.3), np.full(n, 365.0), np.full(n, T, np.int64), method=_native.METHOD_BASELINE, bnd_cap=cap)
db.run(); torch.cuda.synchronize()
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); db.run(); b.record(); torch.cuda.synchronize(); print("ms", a.elapsed_time(b), "cap", cap)
